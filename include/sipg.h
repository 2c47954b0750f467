/* C-ABI of the B200-native SIP-Helmholtz apply (libsipg.so).
 *
 * Replaces the reference's Python operator hot path
 *   HelmholtzOperator.lhs_eval(x) -> y      (reference pkg/src/dgsipg/sipg.py:558-602,
 *                                            alias __call__ at sipg.py:605)
 * whose plan is built by HelmholtzOperator.__init__ (sipg.py:234-281).  The plan
 * descriptor below carries the flattened setup products of that constructor:
 * element classes (sipg.py:302-349), DoF offsets (sipg.py:269-273), geometric
 * factors (mesh.py:331-432), face couplings with transfers, shared-trace rules and
 * penalties (sipg.py:351-554).  It is produced by the Python plan builder
 * (paper_2504_03573_b200/plan.py) and is opaque to callers of sipg_apply.
 *
 * Ownership: the caller owns x / y (device buffers for sipg_apply, host buffers
 * for sipg_apply_host); the plan owns its device tables.  One stream per plan;
 * not re-entrant (like the reference).  All functions return 0 on
 * success or a negative SIPG_ERR_* code; sipg_last_error() describes the last
 * failure on the calling thread.  There is no CPU fallback: without a CUDA
 * device sipg_plan_create fails with SIPG_ERR_NO_DEVICE.
 */
#ifndef SIPG_H
#define SIPG_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SIPG_ERR_ARG (-1)
#define SIPG_ERR_CUDA (-2)
#define SIPG_ERR_NO_DEVICE (-3)
#define SIPG_ERR_UNSUPPORTED (-4)
#define SIPG_ERR_COMM (-5)

typedef struct sipg_plan sipg_plan;

typedef struct sipg_plan_desc {
  int32_t abi_version;      /* must equal the library's SIPG_ABI_VERSION */
  int32_t record_bytes;     /* sizeof(face record) = 128 */
  int32_t dim;              /* 2 or 3 */
  int32_t n_classes;        /* element classes (shape, n_modes, n_quad, geometry) */
  int64_t n_elements;
  int64_t n_dofs;
  int64_t n_records;        /* one per (element, local face) */
  int64_t n_tables, n_elem_geom, n_face_geom;
  double lambda;            /* reaction coefficient (HelmholtzParams.lambda_, sipg.py:64-74) */
  const int32_t* class_desc;   /* n_classes x 64 */
  const int32_t* class_elems;  /* n_elements: element ids grouped by class */
  const int32_t* elem_class;   /* n_elements */
  const int32_t* elem_pos;     /* n_elements: position within its class */
  const int64_t* dof_off;      /* n_elements + 1: element-major DoF offsets (sipg.py:269-273) */
  const void* face_records;    /* n_records x 128 bytes */
  const double* tables;        /* 1-D basis / derivative / transfer tables */
  const double* elem_geom;     /* per-element metric (regular) or per-point (deformed) */
  const double* face_geom;     /* per-face-point swj and G.n where not constant */
  int64_t n_planes;            /* doubles of published face planes (hex), allocated by the plan */
  const int64_t* plane_off;    /* n_elements: offset of each element's 6 face-plane pairs (-1: none) */
  const int64_t* rec_ext;      /* n_records x 2: neighbour face-plane offset | n_o << 48; E tables */
} sipg_plan_desc;

/* Config 4 (3-D hybrid hex / prism / tet; not in the reference): the plan of
 * paper_2504_03573_b200/plan3d.py — element classes (shape, n_modes) with their basis tables,
 * affine element geometry, one 96-byte slot per (element, coupling) (face, trace map, tau,
 * surface Jacobian, metric-normal vector, published-trace offsets).  The same reference
 * interfaces are replaced (HelmholtzOperator.__init__ / lhs_eval, sipg.py:234-281, 558-602);
 * sipg_apply / sipg_apply_host / sipg_cg / sipg_plan_destroy accept the resulting plan. */
typedef struct sipg_h3_desc {
  int32_t abi_version;      /* SIPG_H3_ABI_VERSION of the library (1) */
  int32_t slot_bytes;       /* 96 */
  int32_t n_classes;
  int32_t class_words;      /* 16 int32 per class */
  int64_t n_elements, n_dofs, n_slots, n_tables, n_pub;
  double lambda;
  const int32_t* class_desc;   /* n_classes x 16 */
  const int32_t* class_elems;  /* n_elements: element ids grouped by class */
  const int64_t* dof_off;      /* n_elements + 1 */
  const double* elem_geom;     /* n_elements x 8: |det J|, S = (dxi/dx)(dxi/dx)^T (6), pad */
  const int64_t* slot_off;     /* n_elements + 1: slots of element e are [slot_off[e], slot_off[e+1]) */
  const void* slots;           /* n_slots x 96 bytes */
  const double* tables;        /* basis tables, trace weights, trace maps */
} sipg_h3_desc;
int sipg_h3_plan_create(const sipg_h3_desc* desc, sipg_plan** plan);
/* The flux and apply kernels of a hybrid plan reading `traces` (device, sipg_h3_trace_len doubles, the
 * published-trace layout: per slot (u, n.grad u) per trace point) instead of publishing: with
 * x = 0 and the Dirichlet data as the boundary slots' traces this is the boundary lift of the
 * reference's rhs_assemble (sipg.py:707-717). */
int sipg_h3_apply_traces(sipg_plan* plan, const double* x_dev, const double* traces_dev, double* y_dev,
                         void* stream);
int64_t sipg_h3_trace_len(const sipg_plan* plan);

/* Multi-GPU slab partitions (the paper's trace-only exchange; the
 * reference's stand-in is the in-memory double buffer of sipg.py:565-567 between phase 1 and phase 2).
 * A rank's plan holds its owned elements only; the published traces (u, n.grad u per trace point,
 * sipg.py:585-592) of its partition-face slots are contiguous per neighbour rank (send ranges) and
 * the partner traces arrive in contiguous receive ranges that the slots read directly
 * (paper_2504_03573_b200/halo3d.py builds both orders).  Offsets and counts are in doubles of the
 * published-trace buffer. */
int sipg_h3_set_halo(sipg_plan* plan, int32_t rank, int32_t nranks, int32_t n_nbr, const int32_t* nbr_rank,
                     const int64_t* send_off, const int64_t* send_cnt, const int64_t* recv_off,
                     const int64_t* recv_cnt);
/* NCCL communicator of the partition (ncclCommInitRank with a 128-byte ncclUniqueId that rank 0
 * made with sipg_nccl_unique_id and the caller broadcast): sipg_apply then publishes the
 * boundary-layer traces first, exchanges them with ncclSend / ncclRecv on a high-priority comm
 * stream while the interior elements publish and apply, and applies the boundary layer after the
 * receive.  libnccl.so.2 is resolved at run time (the one torch loaded, if any).  Every element runs
 * the one-GPU arithmetic on the same data, so the owned y is bitwise identical for any rank count. */
int sipg_nccl_unique_id(void* out128);
int sipg_comm_init(sipg_plan* plan, const void* nccl_unique_id, int32_t rank, int32_t nranks);
/* Loop-back transport (tests, one GPU): copy `src`'s send range for dst's rank into dst's receive
 * range for src's rank. */
int sipg_h3_halo_copy(sipg_plan* dst, const sipg_plan* src, void* stream);

/* Build the device-resident plan (uploads all tables). */
int sipg_plan_create(const sipg_plan_desc* desc, sipg_plan** plan);

/* y = (lambda M + L_SIP) x with x, y device pointers of n_dofs doubles, enqueued on
 * `stream` (a cudaStream_t, NULL = legacy default stream).  Replaces lhs_eval. */
int sipg_apply(sipg_plan* plan, const double* x_dev, double* y_dev, void* stream);

/* Only the element classes of one launch role (0: elements whose neighbours are
 * all local, 1: elements touching a ghost element / a partition face, i.e. after
 * the halo exchange; -1: both).  Multi-GPU slabs: role 0, exchange, role 1.
 * Hybrid plans: role 0 publishes every class and applies the interior, role 1
 * applies the boundary layer. */
int sipg_apply_role(sipg_plan* plan, int32_t role, const double* x_dev, double* y_dev, void* stream);

/* One element class only (instrumentation: per-kernel timing).  Classes are
 * independent, so applying every class once equals sipg_apply.  Hybrid 3-D plans
 * (sipg_h3_plan_create) have 3 n_classes launch units, run in this order for a whole apply:
 * every class's publish kernel with the trace maps of its slots (0..n-1), every class's
 * flux launches (2n..3n-1: the per-interface phase 2 of its slots), then every class's
 * apply kernel (n..2n-1). */
int sipg_apply_class(sipg_plan* plan, int32_t cls, const double* x_dev, double* y_dev, void* stream);
/* (shape, n_modes, n_quad, geometry mode, element count, kernel kind) of a class. */
int sipg_plan_class_info(const sipg_plan* plan, int32_t cls, int32_t* out6);

/* Same, from host buffers: H2D copy of x, apply, D2H copy of y, stream sync. */
int sipg_apply_host(sipg_plan* plan, const double* x_host, double* y_host, void* stream);

int sipg_plan_destroy(sipg_plan* plan);

/* GPU-resident unpreconditioned conjugate gradient on A = the plan's operator
 * (reference krylov.cg, pkg/src/dgsipg/krylov.py:39-81):
 * x (device, n doubles, overwritten, starts from 0) approximates A^-1 b (device).
 * maxiter < 0 means the reference default max(10 n, 200); maxiter = 0 runs no iteration
 * (x = 0, reason 4 "maxiter", residual 1).  Same control flow as
 * the reference: stop on p.Ap <= 0 ("indefinite direction", x not updated), on
 * ||r||/||b|| <= tol after verifying the true residual (<= 10 tol, else
 * "residual drift"), on 250 iterations without a 0.1 % improvement
 * ("stagnation"), or at maxiter.  The solver's vectors (r, p, Ap) live in a workspace owned by
 * the plan (allocated by the first solve, reused, freed by sipg_plan_destroy): one solve per plan
 * at a time, like sipg_apply_host's staging buffers. */
typedef struct sipg_solve_report {
  int32_t converged;   /* 1 / 0 */
  int32_t reason;      /* 0 converged, 1 indefinite direction, 2 residual drift, 3 stagnation, 4 maxiter */
  int64_t iterations;
  double residual;     /* relative residual ||b - A x|| / ||b|| (recurrence value unless verified) */
} sipg_solve_report;
int sipg_cg(sipg_plan* plan, const double* b_dev, double* x_dev, int64_t n, double tol, int64_t maxiter,
            sipg_solve_report* report, void* stream);
/* GPU-resident restarted GMRES (reference krylov.gmres, pkg/src/dgsipg/krylov.py:84-141): same
 * interface and stopping rules (restart = max(1, min(restart, n)); converged when the restart
 * residual or the true residual after an update is <= tol; reason 4 "maxiter" otherwise);
 * maxiter < 0 means the reference default max(20 n, 400).  The Arnoldi basis (restart + 1 vectors)
 * lives in the plan's solver workspace; orthogonalisation is classical Gram-Schmidt applied twice
 * (batched multi-dot kernels), one host read per Arnoldi step.  restart <= 255. */
int sipg_gmres(sipg_plan* plan, const double* b_dev, double* x_dev, int64_t n, double tol, int32_t restart,
               int64_t maxiter, sipg_solve_report* report, void* stream);
const char* sipg_last_error(void);

/* Introspection: kernel launches issued so far / per apply; layout constants. */
int64_t sipg_plan_launches(const sipg_plan* plan);
int sipg_plan_kernels_per_apply(const sipg_plan* plan);
int64_t sipg_plan_n_dofs(const sipg_plan* plan);
/* Number of DoF chunks sipg_apply_host pipelines (H2D chunk k || compute stage k-1 || D2H), 0 when
 * the host apply runs copy -> apply -> copy (mesh order not chunkable, or a distributed local plan). */
int sipg_plan_stream_chunks(const sipg_plan* plan);
/* Kernel launches one sipg_apply_host issues (publishers + compute, by stage when streamed). */
int sipg_plan_host_launches_per_apply(const sipg_plan* plan);
int sipg_abi_layout(int32_t* out, int32_t n);
int sipg_supported(int32_t shape, int32_t n_modes, int32_t n_quad);

#ifdef __cplusplus
}
#endif
#endif /* SIPG_H */
