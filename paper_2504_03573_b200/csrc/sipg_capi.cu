// C-ABI of libsipg.so (declared in include/sipg.h).  Plain pointers and sizes:
// no torch types cross this boundary.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>   // types only: libnccl is resolved at run time by sipg_comm_init (dlopen)
#include <stdint.h>
#include <stdio.h>
#include <string.h>
#include <stdlib.h>
#include <string>
#include <vector>
#include "sipg_plan.h"
#include "../../include/sipg.h"
#include "sipg_registry.h"
#include "sipg_h3_registry.h"

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

}  // namespace

void sipg_set_error(const std::string& s) { g_err = s; }   // used by sipg_krylov.cu

namespace {

#define CK(call)                                                                       \
  do {                                                                                 \
    cudaError_t _e = (call);                                                           \
    if (_e != cudaSuccess)                                                             \
      return fail(SIPG_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(_e));  \
  } while (0)

const std::vector<KernelEntry>& kernel_table() {
  static const std::vector<KernelEntry> t = [] {
    std::vector<KernelEntry> v;
    sipg_register_quad(v);
    sipg_register_tri(v);
    sipg_register_hex(v);
    return v;
  }();
  return t;
}

const std::vector<PlanesEntry>& planes_table() {
  static const std::vector<PlanesEntry> t = [] {
    std::vector<PlanesEntry> v;
    sipg_register_planes(v);
    sipg_register_planes_quad(v);
    sipg_register_planes_tri(v);
    return v;
  }();
  return t;
}

const PlanesEntry* find_planes(int shape, int n, int q) {
  for (const auto& k : planes_table())
    if (k.shape == shape && k.n == n && k.q == q) return &k;
  return nullptr;
}

const KernelEntry* find_kernel(int shape, int n, int q, int geom, int kind = 0) {
  for (const auto& k : kernel_table())
    if (k.shape == shape && k.n == n && k.q == q && k.geom == geom && k.kind == kind) return &k;
  return nullptr;
}

// Does every face of every element of class c take the register-column fast
// path (boundary or conforming same-class neighbour, identity transfer,
// constant geometry, no tangential neighbour metric)?  Mirrors k_hex's test.
int class_face_level(const sipg_plan_desc* d, int c) {
  const int32_t* cd = d->class_desc + c * CD_WORDS;
  const FaceRec* recs = (const FaceRec*)d->face_records;
  int level = 0;
  for (int64_t r = cd[CD_REC_OFF]; r < cd[CD_REC_OFF] + (int64_t)cd[CD_COUNT] * cd[CD_NFACES]; ++r) {
    const FaceRec& f = recs[r];
    if (f.type == FT_BOUNDARY && !(f.flags & F_SELF_PW)) continue;
    if (f.type == FT_DIRECT && (f.flags & F_FAST_HEX)) continue;
    if (f.type == FT_SHARED && (f.flags & F_FAST_SHARED) && d->rec_ext && d->rec_ext[2 * r] >= 0) {
      level = 1;
      continue;
    }
    return 2;
  }
  return level;
}

bool class_all_fast(const sipg_plan_desc* d, int c) {
  const int32_t* cd = d->class_desc + c * CD_WORDS;
  const FaceRec* recs = (const FaceRec*)d->face_records;
  for (int64_t r = cd[CD_REC_OFF]; r < cd[CD_REC_OFF] + (int64_t)cd[CD_COUNT] * cd[CD_NFACES]; ++r) {
    const FaceRec& f = recs[r];
    if (f.type == FT_BOUNDARY && !(f.flags & F_SELF_PW)) continue;
    if (f.type == FT_DIRECT && (f.flags & F_FAST_HEX)) continue;
    return false;
  }
  return true;
}

template <typename T>
int upload(const T* host, int64_t count, T** dev) {
  *dev = nullptr;
  if (count <= 0) return 0;
  CK(cudaMalloc((void**)dev, sizeof(T) * count));
  CK(cudaMemcpy(*dev, host, sizeof(T) * count, cudaMemcpyHostToDevice));
  return 0;
}

}  // namespace

// config-4 hybrid hex / prism / tet plan (sipg_h3.cuh)
struct H3State {
  H3Plan hp{};
  std::vector<int32_t> cd;
  std::vector<const H3Entry*> kern;
  std::vector<int> grid_pub, grid_apply;   // persistent grids: min(count, SMs x resident CTAs)
  std::vector<int> cap_pub, cap_apply;     // SMs x resident CTAs
  // register-column kernels: own-grid fluxes per slot, written by the flux kernel (one warp per slot,
  // work list cslots = slot ids in class-list order; cslot_off[i] = first entry of class-list position i)
  bool flux = false;
  double* fb = nullptr;
  int64_t* fb_off_d = nullptr;
  H3FluxRec* frec_d = nullptr;
  double* ug = nullptr;          // u on the q^3 grids, publish -> apply
  int64_t* ug_off_d = nullptr;
  long long* escal_d = nullptr;  // per class-list position: element scalars (H3Plan::escal)
  std::vector<int64_t> cs_id, cs_mp;   // per class-list position: first identity-map / mapped record
  int64_t n_id = 0;                    // records: [identity-map slots | mapped slots], each in class-list order
  // streamed host apply (see build_stream_schedule_h3): per stage, publish rows and apply rows
  struct Launch { int row, grid; const H3Entry* k; int pos0, pos1; };   // pos: class-list positions of the row
  std::vector<std::vector<Launch>> st_pub, st_comp;
  int32_t* rows_d = nullptr;
  H3Plan hps{};
  // streamed host apply: the slot records once more, ordered by stage (one trace-map launch and two flux
  // launches per stage instead of three per class row): per stage k the ranges [st_mp[k], st_mp[k+1]) etc.
  H3FluxRec* frec_stage_d = nullptr;
  std::vector<int64_t> st_mp, st_fi, st_fm;
  std::vector<H3FluxRec> frec_host;   // kept until the stream schedule is built
  void* bufs[7] = {};
  double* pub = nullptr;
  int64_t n_pub = 0;
  // trace halo of a slab partition (sipg_h3_set_halo): per neighbour rank the published-trace
  // ranges (doubles) this rank sends and the ones it receives; NCCL point-to-point over NVLink on
  // a dedicated stream (sipg_comm_init)
  int rank = -1, nranks = 0;
  std::vector<int32_t> nbr;
  std::vector<int64_t> send_off, send_cnt, recv_off, recv_cnt;
  ncclComm_t comm = nullptr;
  cudaStream_t s_comm = nullptr;
  cudaEvent_t ev_pub1 = nullptr, ev_comm = nullptr;
  bool fork_all = false;
};

// Independent class launches (the publishers of a phase, then the element classes) are spread over
// the caller's stream and a few side streams, forked / joined with events, when at least two of
// them are too small to fill the GPU (grid below SMs x resident CTAs): such classes then run side by
// side instead of one after another (cfg1: 0.121 -> 0.081 ms).  Full-size persistent launches gain
// nothing from it (measured on cfg2 / cfg3b / cfg4) and skip the fork.  SIPG_CONCURRENT=0 disables
// it (instrumentation).
struct Fork {
  std::vector<cudaStream_t> side;
  cudaEvent_t ev_fork = nullptr;
  std::vector<cudaEvent_t> ev_join;
  int next = 0;       // round-robin position inside the current group
  int used = 0;       // side streams used by the current group
  cudaStream_t s = nullptr;
};

struct sipg_plan {
  H3State* h3 = nullptr;
  Fork fork;
  DevPlan dp;
  int n_cls;
  int64_t n_dofs;
  std::vector<int32_t> cd_host;
  std::vector<const KernelEntry*> kern;
  std::vector<int> grid;                 // CTAs per class launch (persistent kernels: SMs x occupancy)
  std::vector<const PlanesEntry*> planes_k;   // per class: face-plane publisher (hex) or null
  bool need_planes = false;
  double* planes = nullptr;
  void* bufs[11];
  double* x_stage = nullptr;
  double* y_stage = nullptr;
  // solver workspace (sipg_cg): device vectors + reduction scratch and pinned scalars, kept across
  // solves (allocated on first use, grown on demand, freed with the plan)
  void* ws = nullptr;
  size_t ws_bytes = 0;
  double* ws_host = nullptr;
  size_t ws_host_n = 0;
  int64_t launches = 0;
  std::vector<int> per_sm;               // resident CTAs per SM of each class's kernel
  struct Graph { const double* x; double* y; cudaGraphExec_t exec; int64_t kernels; };
  std::vector<Graph> graphs;             // captured whole applies (sipg_apply)
  struct HostGraph { const double* x; double* y; cudaGraphExec_t exec; int64_t kernels; };
  std::vector<HostGraph> host_graphs;    // captured streamed host applies (sipg_apply_host)
  bool use_graphs = true;
  cudaStream_t cap_stream = nullptr;
  int sms = 0;                           // multiprocessors of the plan's device (queried)
  bool stream_trace = false;             // SIPG_STREAM_TRACE, read once at plan creation
  // Streamed host apply (sipg_apply_host): x is copied H2D in K DoF chunks; chunk k's elements
  // publish their planes/traces as soon as it lands, and the elements whose neighbourhood lies in
  // chunks <= k ("stage k") compute right after; y chunks go back D2H as soon as their last stage
  // is done.  The rows are sub-ranges of the class lists (classes are in ascending element order),
  // so the kernels run unchanged on a second descriptor array.
  struct Launch { int row, grid; const KernelEntry* k; const PlanesEntry* pe; };
  bool streamed = false;
  int n_chunks = 0;
  std::vector<int64_t> chunk_dof;        // K + 1 dof boundaries
  std::vector<std::vector<Launch>> pub, comp;
  std::vector<int> d2h_stage;            // per chunk: the stage after which its y is complete
  DevPlan dps{};
  int32_t* cds_d = nullptr;
  cudaStream_t s_h2d = nullptr, s_d2h = nullptr;
  std::vector<cudaEvent_t> ev_h2d, ev_comp;
  cudaEvent_t ev_start = nullptr, ev_done = nullptr;
};

namespace {

constexpr int kSideStreams = 3;

// element count below which a 2-D class runs CTA-per-element (SIPG_SMALL_CLASS overrides)
int small_class_elems() {
  static const int v = [] {
    const char* e = getenv("SIPG_SMALL_CLASS");
    return e ? atoi(e) : 512;   // cfg0 (256 elements) 24.6 -> 22.5 us; cfg1 classes (~1000) are faster per warp
  }();
  return v;
}

// Instrumentation switches that change results exist only in SIPG_INSTRUMENT builds
// (build.py OUT.so -DSIPG_INSTRUMENT); the product library ignores them.
int instrument_debug() {
#ifdef SIPG_INSTRUMENT
  const char* e = getenv("SIPG_DEBUG");
  return e ? atoi(e) : 0;
#else
  return 0;
#endif
}

bool concurrency_on() {
  static const bool on = [] {
    const char* e = getenv("SIPG_CONCURRENT");
    return !(e && atoi(e) == 0);
  }();
  return on;
}

// begin a group of independent launches on s; returns the stream for launch i via group_stream
int fork_create(sipg_plan* p) {
  Fork& f = p->fork;
  if (f.side.empty()) {
    f.side.resize(kSideStreams);
    f.ev_join.resize(kSideStreams);
    for (int j = 0; j < kSideStreams; ++j) {
      if (cudaStreamCreateWithFlags(&f.side[j], cudaStreamNonBlocking) != cudaSuccess ||
          cudaEventCreateWithFlags(&f.ev_join[j], cudaEventDisableTiming) != cudaSuccess)
        return fail(SIPG_ERR_CUDA, "side stream / event creation");
    }
    if (cudaEventCreateWithFlags(&f.ev_fork, cudaEventDisableTiming) != cudaSuccess)
      return fail(SIPG_ERR_CUDA, "fork event creation");
  }
  return 0;
}

int group_begin(sipg_plan* p, cudaStream_t s, int nlaunch, int nsmall) {
  Fork& f = p->fork;
  f.s = s;
  f.next = 0;
  f.used = 0;
  if (nlaunch <= 1 || nsmall < 2 || !concurrency_on()) return 0;
  if (int rc = fork_create(p)) return rc;
  f.used = nlaunch - 1 < kSideStreams ? nlaunch - 1 : kSideStreams;
  CK(cudaEventRecord(f.ev_fork, s));
  for (int j = 0; j < f.used; ++j) CK(cudaStreamWaitEvent(f.side[j], f.ev_fork, 0));
  return 0;
}

cudaStream_t group_stream(sipg_plan* p) {
  Fork& f = p->fork;
  if (f.used == 0) return f.s;
  const int i = f.next++ % (f.used + 1);
  return i == 0 ? f.s : f.side[i - 1];
}

int group_end(sipg_plan* p) {
  Fork& f = p->fork;
  for (int j = 0; j < f.used; ++j) {
    CK(cudaEventRecord(f.ev_join[j], f.side[j]));
    CK(cudaStreamWaitEvent(f.s, f.ev_join[j], 0));
  }
  f.used = 0;
  return 0;
}

__global__ void k_stamp(unsigned long long* buf, int i) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  buf[i] = t;
}

int launch_grid(const KernelEntry* k, int count, int per_sm, int sms) {
  if (k->kind == 0) return count;   // CTA per element
  const int epc = k->kind == 5 ? k->threads / 32 : 1;   // warp-per-element kernels
  const int g = (count + epc - 1) / epc;
  return g < per_sm * sms ? g : per_sm * sms;
}

int publish_grid(const int32_t* cd, int count, int sms) {
  const int per = cd[CD_SHAPE] == SHAPE_HEX ? 1 : 8;
  const int g = (count + per - 1) / per;
  return g < sms * 8 ? g : sms * 8;
}

// DoF chunk boundaries of the streamed host apply (4 KB-aligned).  Graduated chunks: quarter- and
// half-size chunks at both ends (1 2 4 4 ... 4 2 1 in units of chunk_bytes / 4), so that the compute
// starts after a short first copy and the copies of the y chunks the last stage completes are short
// (measured on cfg4 with uniform 24 MB chunks: 0.5 ms before the first stage, 0.9 ms of D2H after
// the last one; host apply 9.0 -> 8.1 ms with the graduated chunks and graph replay).
// SIPG_STREAM_UNIFORM=1 keeps uniform chunks.  Returns K (0: too small to stream).
int make_chunks(sipg_plan* p, int64_t ndof, int64_t chunk_bytes) {
  const double units = (double)ndof * 8 / (chunk_bytes > 0 ? chunk_bytes : 1) * 4.0;
  auto place = [&](std::vector<double> w) -> int {
    int K = (int)w.size();
    if (K > 64) K = 64;
    if (K < 2) return 0;
    w.resize(K);
    p->chunk_dof.assign(K + 1, 0);
    double tot = 0.0, acc = 0.0;
    for (double v : w) tot += v;
    for (int k = 1; k < K; ++k) {
      acc += w[k - 1];
      p->chunk_dof[k] = (int64_t)((double)ndof * acc / tot) & ~(int64_t)511;
    }
    p->chunk_dof[K] = ndof;
    for (int k = 0; k < K; ++k)
      if (p->chunk_dof[k + 1] <= p->chunk_dof[k]) return 0;
    return K;
  };
  if (!getenv("SIPG_STREAM_UNIFORM") && units >= 16) {   // graduated: short first copy, short tail
    std::vector<double> w = {1, 2};
    const int mid = (int)((units - 6) / 4 + 0.5);
    for (int k = 0; k < mid; ++k) w.push_back(4);
    w.push_back(2);
    w.push_back(1);
    const int K = place(w);
    if (K) return K;   // else (4 KB alignment leaves a short chunk empty on small meshes): uniform chunks
  }
  return place(std::vector<double>((size_t)(units / 4 > 0 ? units / 4 : 0), 1.0));
}

// Build the streamed-apply schedule (see sipg_plan).  Returns false when the mesh ordering does not
// allow it (a class whose element list is not monotone in stage) — the host apply then runs
// copy -> apply -> copy.
bool build_stream_schedule(sipg_plan* p, const sipg_plan_desc* d) {
  const int64_t nel = d->n_elements, ndof = d->n_dofs;
  const int64_t bytes = ndof * 8;
  // chunk size: >= 12 MB (~0.22 ms of PCIe), and >= 1.5 MB per launch a stage issues (per-class
  // stage launches get short and tail-bound on multi-class meshes; measured on cfg3a / cfg3b).
  // Measured and rejected: kernels storing y straight into page-locked host memory (no D2H
  // copies) — equal on cfg3a, 13 % slower on cfg3b, even with whole-warp y stores.
  // SIPG_STREAM_CHUNK_BYTES overrides (tests use small meshes)
  int launches_per_stage = 0;
  for (int c = 0; c < d->n_classes; ++c)
    if (d->class_desc[c * CD_WORDS + CD_COUNT] > 0) launches_per_stage += p->planes_k[c] ? 2 : 1;
  int64_t chunk_bytes = (int64_t)launches_per_stage * (3ll << 19);
  if (chunk_bytes < (12ll << 20)) chunk_bytes = 12ll << 20;
  // mid-size meshes (16-48 MB of x): two chunks still overlap half of each copy direction with the
  // compute (cfg2, 22.6 MB: host apply 2.21 -> 2.03 ms)
  if (bytes >= (16ll << 20) && chunk_bytes > bytes / 2) chunk_bytes = bytes / 2 - 4096;
  const char* cb = getenv("SIPG_STREAM_CHUNK_BYTES");
  if (cb) chunk_bytes = atoll(cb);
  for (int c = 0; c < d->n_classes; ++c)
    if (d->class_desc[c * CD_WORDS + CD_ROLE] != 0) return false;   // distributed local plans: no
  // copy chunks: 4 KB-aligned DoF ranges (DMA runs markedly slower on unaligned host ranges when
  // both directions are busy); an element belongs to the chunk in which its last DoF arrives
  const int K = make_chunks(p, ndof, chunk_bytes);
  if (K < 2) return false;
  std::vector<int32_t> chunk(nel), stage(nel);
  {
    int k = 0;
    for (int64_t e = 0; e < nel; ++e) {
      while (d->dof_off[e + 1] > p->chunk_dof[k + 1]) ++k;
      chunk[e] = k;
    }
  }
  const FaceRec* recs = (const FaceRec*)d->face_records;
  for (int c = 0; c < d->n_classes; ++c) {
    const int32_t* cd = d->class_desc + c * CD_WORDS;
    const int nf = cd[CD_NFACES];
    for (int i = 0; i < cd[CD_COUNT]; ++i) {
      const int el = d->class_elems[cd[CD_ELEM_OFF] + i];
      int st = chunk[el];
      for (int f = 0; f < nf; ++f) {
        const int nb = recs[(int64_t)cd[CD_REC_OFF] + (int64_t)i * nf + f].nbr;
        if (nb >= 0 && chunk[nb] > st) st = chunk[nb];
      }
      // an element may run later than its neighbourhood allows: keep stages monotone along the
      // class list so each stage is one contiguous sub-range of it
      if (i > 0 && stage[d->class_elems[cd[CD_ELEM_OFF] + i - 1]] > st) st = stage[d->class_elems[cd[CD_ELEM_OFF] + i - 1]];
      stage[el] = st;
    }
  }
  // rows are appended after the original classes: kernels look neighbours' classes up by
  // elem_class in the same descriptor array
  std::vector<int32_t> rows(d->class_desc, d->class_desc + (int64_t)d->n_classes * CD_WORDS);
  p->pub.assign(K, {});
  p->comp.assign(K, {});
  p->d2h_stage.assign(K, 0);
  {   // y range j is complete once every element overlapping it has run
    int j = 0;
    for (int64_t el = 0; el < nel; ++el) {
      while (d->dof_off[el] >= p->chunk_dof[j + 1]) ++j;
      for (int jj = j; jj < K && p->chunk_dof[jj] < d->dof_off[el + 1]; ++jj)
        if (stage[el] > p->d2h_stage[jj]) p->d2h_stage[jj] = stage[el];
    }
  }
  auto add_row = [&](const int32_t* cd, int i0, int i1) {
    const int r = (int)(rows.size() / CD_WORDS);
    rows.insert(rows.end(), cd, cd + CD_WORDS);
    int32_t* w = rows.data() + (int64_t)r * CD_WORDS;
    w[CD_COUNT] = i1 - i0;
    w[CD_ELEM_OFF] += i0;
    w[CD_REC_OFF] += i0 * cd[CD_NFACES];
    w[CD_EGEO_OFF] += i0 * cd[CD_EGEO_STRIDE];
    return r;
  };
  for (int c = 0; c < d->n_classes; ++c) {
    const int32_t* cd = d->class_desc + c * CD_WORDS;
    const int n = cd[CD_COUNT];
    const int32_t* el = d->class_elems + cd[CD_ELEM_OFF];
    for (int pass = 0; pass < 2; ++pass) {   // 0: publisher rows by chunk, 1: compute rows by stage
      if (pass == 0 && !p->planes_k[c]) continue;
      const std::vector<int32_t>& key = pass == 0 ? chunk : stage;
      int i0 = 0;
      while (i0 < n) {
        const int k = key[el[i0]];
        int i1 = i0;
        while (i1 < n && key[el[i1]] == k) ++i1;
        for (int j = i1; j < n; ++j)
          if (key[el[j]] <= k) return false;   // not monotone: no streaming
        const int r = add_row(cd, i0, i1);
        if (pass == 0)
          p->pub[k].push_back({r, publish_grid(cd, i1 - i0, p->sms), nullptr, p->planes_k[c]});
        else
          p->comp[k].push_back({r, launch_grid(p->kern[c], i1 - i0, p->per_sm[c], p->sms), p->kern[c], nullptr});
        i0 = i1;
      }
    }
  }
  if (upload(rows.data(), (int64_t)rows.size(), &p->cds_d)) return false;
  p->dps = p->dp;
  p->dps.cd = p->cds_d;
  p->n_chunks = K;
  return true;
}

}  // namespace

extern "C" {

const char* sipg_last_error(void) { return g_err.c_str(); }

int sipg_abi_layout(int32_t* out, int32_t n) {
  const int32_t v[] = {SIPG_ABI_VERSION, (int32_t)sizeof(FaceRec), CD_WORDS, CD_TAX, TR_GSTART,
                       F_OTHER_NEG, (int32_t)offsetof(FaceRec, tau), (int32_t)offsetof(FaceRec, gs)};
  const int m = (int)(sizeof(v) / sizeof(v[0]));
  for (int i = 0; i < n && i < m; ++i) out[i] = v[i];
  return m;
}

int sipg_supported(int32_t shape, int32_t n_modes, int32_t n_quad) {
  return find_kernel(shape, n_modes, n_quad, GEOM_REGULAR, shape == SHAPE_HEX ? 0 : 5) != nullptr;
}

int sipg_plan_create(const sipg_plan_desc* d, sipg_plan** out) {
  if (!d || !out) return fail(SIPG_ERR_ARG, "null argument");
  *out = nullptr;
  if (d->abi_version != SIPG_ABI_VERSION)
    return fail(SIPG_ERR_ARG, "ABI version mismatch: plan built for " + std::to_string(d->abi_version) +
                                  ", library is " + std::to_string(SIPG_ABI_VERSION));
  if (d->record_bytes != (int32_t)sizeof(FaceRec)) return fail(SIPG_ERR_ARG, "face record size mismatch");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return fail(SIPG_ERR_NO_DEVICE, "no CUDA device available (the SIP apply has no CPU fallback)");
  sipg_plan* p = new sipg_plan();
  memset(p->bufs, 0, sizeof(p->bufs));
  p->n_cls = d->n_classes;
  p->n_dofs = d->n_dofs;
  p->cd_host.assign(d->class_desc, d->class_desc + (int64_t)d->n_classes * CD_WORDS);
  for (int c = 0; c < d->n_classes; ++c) {
    const int32_t* cd = d->class_desc + c * CD_WORDS;
    const int shape = cd[CD_SHAPE], n = cd[CD_N], q = cd[CD_Q0], geom = cd[CD_GEOM];
    bool uniform = true;
    const int dim = shape == SHAPE_HEX ? 3 : 2;
    for (int a = 1; a < dim; ++a) uniform = uniform && cd[CD_Q0 + a] == q;
    const KernelEntry* k = nullptr;
    if (uniform && shape == SHAPE_HEX && geom == GEOM_REGULAR && cd[CD_KIND] == 0 && cd[CD_GLLMASK] == 7 &&
        !getenv("SIPG_GENERIC_KERNELS")) {
      // all faces boundary / conforming-fast: k_hex (kind 4); fast shared traces: k_hexp (kind 7);
      // anything else: k_hex with the generic face path (kind 2)
      const int level = class_face_level(d, c);
      k = find_kernel(shape, n, q, geom, level == 0 ? 4 : (level == 1 ? 7 : 2));
      if (k) {
        const int* ax = cd + CD_TAX;
        cudaError_t e = k->upload(d->tables + ax[TX_V], d->tables + ax[TX_D], d->tables + ax[TX_W],
                                  d->tables + ax[TX_DVEND]);
        if (e != cudaSuccess) {
          sipg_plan_destroy(p);
          return fail(SIPG_ERR_CUDA, std::string("constant table upload: ") + cudaGetErrorString(e));
        }
      }
    }
    if (!k && uniform) k = find_kernel(shape, n, q, geom, shape == SHAPE_HEX ? 0 : 5);
    // 2-D classes too small to fill the GPU with warp-per-element pipelines: one CTA per element
    // (every element in flight at once; the per-element latency, not throughput, is the cost)
    if (k && k->kind == 5 && cd[CD_COUNT] <= small_class_elems()) {
      const KernelEntry* kc = find_kernel(shape, n, q, geom, 0);
      if (kc) k = kc;
    }
    if (!k) {
      sipg_plan_destroy(p);
      return fail(SIPG_ERR_UNSUPPORTED, "no sm_100a kernel for shape=" + std::to_string(shape) +
                                            " n_modes=" + std::to_string(n) + " n_quad=" + std::to_string(q));
    }
    p->kern.push_back(k);
  }
  // every device buffer is owned by p->bufs from the moment it exists, so any failure below can
  // release the partial plan through sipg_plan_destroy
  int rc = 0;
  int nb = 0;
  auto up = [&](const auto* host, int64_t count, auto** dev) -> int {
    int r = upload(host, count, dev);
    p->bufs[nb++] = (void*)*dev;
    return r;
  };
  int32_t *cd_d, *ce_d, *ec_d, *ep_d;
  int64_t* dof_d;
  FaceRec* rec_d;
  double *tab_d, *eg_d, *fg_d;
  int64_t *po_d = nullptr, *rx_d = nullptr;
  if ((rc = up(d->class_desc, (int64_t)d->n_classes * CD_WORDS, &cd_d)) ||
      (rc = up(d->class_elems, d->n_elements, &ce_d)) || (rc = up(d->elem_class, d->n_elements, &ec_d)) ||
      (rc = up(d->elem_pos, d->n_elements, &ep_d)) || (rc = up(d->dof_off, d->n_elements + 1, &dof_d)) ||
      (rc = up((const FaceRec*)d->face_records, d->n_records, &rec_d)) ||
      (rc = up(d->tables, d->n_tables, &tab_d)) || (rc = up(d->elem_geom, d->n_elem_geom, &eg_d)) ||
      (rc = up(d->face_geom, d->n_face_geom, &fg_d)) ||
      (rc = up(d->plane_off, d->plane_off ? d->n_elements : 0, &po_d)) ||
      (rc = up(d->rec_ext, d->rec_ext ? 2 * d->n_records : 0, &rx_d))) {
    sipg_plan_destroy(p);
    return rc;
  }
  // Published neighbour data: hex planes for the k_hexp classes; 2-D face traces when the mesh has
  // triangles (a triangle trace costs a collapsed-coordinate chain per face — worth computing once per
  // face instead of once per reader; quad traces are cheap enough to evaluate in place).
  for (const KernelEntry* k : p->kern)
    p->need_planes = p->need_planes || k->kind == 6 || k->kind == 7 || (k->kind == 5 && k->shape == SHAPE_TRI);
  if (getenv("SIPG_NO_PUBLISH")) p->need_planes = false;   // instrumentation: 2-D kernels evaluate neighbours
  if (p->need_planes && d->n_planes > 0) {
    cudaError_t e = cudaMalloc((void**)&p->planes, sizeof(double) * d->n_planes);
    if (e != cudaSuccess) {
      p->planes = nullptr;
      sipg_plan_destroy(p);
      return fail(SIPG_ERR_CUDA, std::string("face-plane buffer: ") + cudaGetErrorString(e));
    }
  }
  for (int c = 0; c < d->n_classes; ++c) {
    const int32_t* cd = d->class_desc + c * CD_WORDS;
    const PlanesEntry* pe = nullptr;
    if (p->need_planes && cd[CD_SHAPE] != SHAPE_HEX) {
      pe = find_planes(cd[CD_SHAPE], cd[CD_N], cd[CD_Q0]);
      if (!pe) {
        sipg_plan_destroy(p);
        return fail(SIPG_ERR_UNSUPPORTED, "no face-trace publisher for this 2-D class");
      }
    } else if (p->need_planes && cd[CD_SHAPE] == SHAPE_HEX && cd[CD_KIND] == 0 && cd[CD_GLLMASK] == 7) {
      pe = find_planes(SHAPE_HEX, cd[CD_N], cd[CD_Q0]);
      const int* ax = cd + CD_TAX;
      const KernelEntry* kf = find_kernel(SHAPE_HEX, cd[CD_N], cd[CD_Q0], GEOM_REGULAR, 4);
      if (pe && kf) {   // the publisher reads the (N, Q) constant tables
        cudaError_t e = kf->upload(d->tables + ax[TX_V], d->tables + ax[TX_D], d->tables + ax[TX_W],
                                   d->tables + ax[TX_DVEND]);
        if (e != cudaSuccess) {
          sipg_plan_destroy(p);
          return fail(SIPG_ERR_CUDA, std::string("constant table upload: ") + cudaGetErrorString(e));
        }
      }
      if (!pe) {
        sipg_plan_destroy(p);
        return fail(SIPG_ERR_UNSUPPORTED, "no face-plane publisher for this hex class");
      }
    }
    p->planes_k.push_back(pe);
  }
  p->dp = DevPlan{cd_d, ce_d, ec_d, ep_d, dof_d, rec_d, tab_d, eg_d, fg_d, d->lambda, d->dim, d->n_classes,
                  instrument_debug(), 0, p->planes, po_d, rx_d};
  for (const KernelEntry* k : p->kern) {
    if (k->smem == 0) continue;
    cudaError_t e = cudaFuncSetAttribute((const void*)k->fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)k->smem);
    if (e != cudaSuccess) {
      sipg_plan_destroy(p);
      return fail(SIPG_ERR_CUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
    }
  }
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0) {
    sipg_plan_destroy(p);
    return fail(SIPG_ERR_CUDA, "multiprocessor count query failed");
  }
  p->sms = sms;
  p->stream_trace = getenv("SIPG_STREAM_TRACE") != nullptr;
  p->use_graphs = !getenv("SIPG_NO_GRAPH");
  for (int c = 0; c < p->n_cls; ++c) {
    const KernelEntry* k = p->kern[c];
    const int count = p->cd_host[c * CD_WORDS + CD_COUNT];
    int per_sm = 1;
    if (k->kind != 0) {
      cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void*)k->fn, k->threads, k->smem);
      if (e != cudaSuccess || per_sm <= 0) {
        sipg_plan_destroy(p);
        return fail(SIPG_ERR_CUDA, "occupancy query failed for a persistent kernel");
      }
    }
    p->per_sm.push_back(per_sm);
    p->grid.push_back(launch_grid(k, count, p->per_sm.back(), sms));
  }
  p->streamed = !getenv("SIPG_NO_STREAM") && build_stream_schedule(p, d);
  *out = p;
  return 0;
}

// ---------------------------------------------------------------------------------------------
// NCCL, resolved at run time (the library loads without it; torch's own libnccl.so.2 is reused
// when already loaded in the process)
struct NcclApi {
  bool ok = false;
  std::string err;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*commGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
  const char* (*errorString)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    const char* env = getenv("SIPG_NCCL_LIB");
    if (!h && env) h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      a.err = "libnccl.so.2 not found (import torch first, or set SIPG_NCCL_LIB)";
      return a;
    }
    auto sym = [&](auto& fp, const char* name) { fp = reinterpret_cast<std::decay_t<decltype(fp)>>(dlsym(h, name)); };
    sym(a.getUniqueId, "ncclGetUniqueId");
    sym(a.commInitRank, "ncclCommInitRank");
    sym(a.commDestroy, "ncclCommDestroy");
    sym(a.commGetAsyncError, "ncclCommGetAsyncError");
    sym(a.send, "ncclSend");
    sym(a.recv, "ncclRecv");
    sym(a.groupStart, "ncclGroupStart");
    sym(a.groupEnd, "ncclGroupEnd");
    sym(a.errorString, "ncclGetErrorString");
    a.ok = a.getUniqueId && a.commInitRank && a.commDestroy && a.commGetAsyncError && a.send && a.recv &&
           a.groupStart && a.groupEnd && a.errorString;
    if (!a.ok) a.err = "libnccl.so.2 lacks a required symbol";
    return a;
  }();
  return api;
}

#define NCK(call)                                                                                   \
  do {                                                                                              \
    ncclResult_t _r = (call);                                                                       \
    if (_r != ncclSuccess) return fail(SIPG_ERR_COMM, std::string(#call) + ": " + nccl().errorString(_r)); \
  } while (0)

// the slot kernels (pass 2 flux, 3 trace maps) over the class-list positions [a, b): identity-map and
// mapped slots are separate work lists (uniform warps per launch)
static void h3_slot_launch(sipg_plan* p, const H3Plan& hp, int pass, int a, int b, cudaStream_t s) {
  H3State* h = p->h3;
  const int64_t i0 = h->cs_id[a], i1 = h->cs_id[b], m0 = h->n_id + h->cs_mp[a], m1 = h->n_id + h->cs_mp[b];
  if (pass == 2) {
    if (i1 > i0) { sipg_h3c_flux_launch(hp, i0, i1 - i0, false, p->sms, s); ++p->launches; }
    if (m1 > m0) { sipg_h3c_flux_launch(hp, m0, m1 - m0, true, p->sms, s); ++p->launches; }
  } else if (m1 > m0) {
    sipg_h3c_map_launch(hp, m0, m1 - m0, p->sms, s);
    ++p->launches;
  }
}

// launch the classes of one pass (0 publish, 1 apply, 2 flux: the slots of those classes, adjacent
// classes merged into one launch) whose role is selected by `want` (-1: all)
int h3_launch(sipg_plan* p, int pass, int want, const double* x_dev, double* y_dev, cudaStream_t s) {
  H3State* h = p->h3;
  auto go = [&](int c) {
    const int count = h->cd[c * CD3_WORDS + CD3_COUNT];
    const int crole = h->cd[c * CD3_WORDS + CD3_ROLE];
    return count > 0 && (want < 0 || crole == want);
  };
  if (pass >= 2) {   // 2 flux, 3 trace maps: the slots of the selected classes, adjacent classes merged
    if (!h->flux) return 0;
    int c0 = -1;
    for (int c = 0; c <= p->n_cls; ++c) {
      const bool on = c < p->n_cls && go(c);
      if (on && c0 < 0) c0 = c;
      if (!on && c0 >= 0) {
        const int a = h->cd[c0 * CD3_WORDS + CD3_ELEM_OFF];
        const int b = h->cd[(c - 1) * CD3_WORDS + CD3_ELEM_OFF] + h->cd[(c - 1) * CD3_WORDS + CD3_COUNT];
        h3_slot_launch(p, h->hp, pass, a, b, s);
        c0 = -1;
      }
    }
    return 0;
  }
  int n = 0, nsmall = 0;
  for (int c = 0; c < p->n_cls; ++c) {
    if (!go(c)) continue;
    ++n;
    nsmall += (pass == 0 ? h->grid_pub[c] < h->cap_pub[c] : h->grid_apply[c] < h->cap_apply[c]);
  }
  if (h->fork_all) nsmall = n;   // SIPG_H3_FORK=1: run even full-size class launches side by side
  int rc = group_begin(p, s, n, nsmall);
  if (rc) return rc;
  for (int c = 0; c < p->n_cls; ++c) {
    if (!go(c)) continue;
    const H3Entry* k = h->kern[c];
    cudaStream_t st = group_stream(p);
    if (pass == 0)
      k->pub<<<h->grid_pub[c], k->threads, k->smem_pub, st>>>(h->hp, c, x_dev, y_dev);
    else
      k->apply<<<h->grid_apply[c], k->threads, k->smem_apply, st>>>(h->hp, c, x_dev, y_dev);
    ++p->launches;
  }
  return group_end(p);
}

// Trace-halo exchange of a partitioned plan on the comm stream: every neighbour's send range of the
// published traces goes out and its range arrives in this rank's receive region, one NCCL group.
int h3_exchange(sipg_plan* p) {
  H3State* h = p->h3;
  const NcclApi& a = nccl();
  NCK(a.groupStart());
  for (size_t i = 0; i < h->nbr.size(); ++i) {
    if (h->send_cnt[i] > 0)
      NCK(a.send(h->pub + h->send_off[i], (size_t)h->send_cnt[i], ncclFloat64, h->nbr[i], h->comm, h->s_comm));
    if (h->recv_cnt[i] > 0)
      NCK(a.recv(h->pub + h->recv_off[i], (size_t)h->recv_cnt[i], ncclFloat64, h->nbr[i], h->comm, h->s_comm));
  }
  NCK(a.groupEnd());
  return 0;
}

// The apply of a hybrid plan.  Whole plan (role -1): publish the boundary-layer classes (role 1)
// first; with a trace halo and a communicator, their traces leave on the comm stream while the
// interior classes (role 0) publish and apply; the boundary-layer classes apply once the partner
// traces have arrived.  role 0 / 1 (a caller-driven exchange between them): 0 publishes every class
// and applies the interior, 1 applies the boundary layer.
int h3_apply(sipg_plan* p, int role, const double* x_dev, double* y_dev, cudaStream_t s) {
  H3State* h = p->h3;
  int rc = 0;
  // pass 0 publish, 3 trace maps, 2 flux, 1 apply
  if (role == 1) {
    if ((rc = h3_launch(p, 2, 1, x_dev, y_dev, s))) return rc;
    if ((rc = h3_launch(p, 1, 1, x_dev, y_dev, s))) return rc;
    CK(cudaGetLastError());
    return 0;
  }
  const bool halo = h->nranks > 1 && !h->nbr.empty();
  if (role < 0 && halo && !h->comm)
    return fail(SIPG_ERR_ARG, "partitioned plan without a communicator: call sipg_comm_init, or drive the "
                              "exchange with sipg_apply_role 0 / 1");
  if ((rc = h3_launch(p, 0, 1, x_dev, y_dev, s))) return rc;     // boundary layer publishes first
  if ((rc = h3_launch(p, 3, 1, x_dev, y_dev, s))) return rc;
  if (role < 0 && halo) {
    ncclResult_t ae = ncclSuccess;
    if (nccl().commGetAsyncError(h->comm, &ae) != ncclSuccess || ae != ncclSuccess)
      return fail(SIPG_ERR_COMM, std::string("NCCL asynchronous error: ") + nccl().errorString(ae));
    CK(cudaEventRecord(h->ev_pub1, s));
    CK(cudaStreamWaitEvent(h->s_comm, h->ev_pub1, 0));
    if ((rc = h3_exchange(p))) return rc;
    CK(cudaEventRecord(h->ev_comm, h->s_comm));
  }
  if ((rc = h3_launch(p, 0, 0, x_dev, y_dev, s))) return rc;
  if ((rc = h3_launch(p, 3, 0, x_dev, y_dev, s))) return rc;
  if ((rc = h3_launch(p, 2, 0, x_dev, y_dev, s))) return rc;
  if ((rc = h3_launch(p, 1, 0, x_dev, y_dev, s))) return rc;
  if (role < 0) {
    if (halo) CK(cudaStreamWaitEvent(s, h->ev_comm, 0));
    if ((rc = h3_launch(p, 2, 1, x_dev, y_dev, s))) return rc;
    if ((rc = h3_launch(p, 1, 1, x_dev, y_dev, s))) return rc;
  }
  CK(cudaGetLastError());
  return 0;
}

// Streamed host apply for hybrid plans: x arrives in 4 KB-aligned DoF chunks; as chunk k lands, its
// elements publish their traces, and the elements whose partners all lie in chunks <= k ("stage k")
// apply; y chunks go back as soon as their last stage is done (same pipeline as the standard plans,
// build_stream_schedule).  Rows are sub-ranges of the class lists appended after the classes.
bool build_stream_schedule_h3(sipg_plan* p, const sipg_h3_desc* d) {
  H3State* h = p->h3;
  const int64_t nel = d->n_elements, ndof = d->n_dofs;
  int launches_per_stage = 0;
  for (int c = 0; c < d->n_classes; ++c) {
    if (d->class_desc[c * CD3_WORDS + CD3_ROLE] != 0) return false;    // distributed local plans: no
    if (d->class_desc[c * CD3_WORDS + CD3_COUNT] > 0) launches_per_stage += 2;
  }
  // 24 MB chunks (the stage rows run side by side, so short launches cost little; measured on cfg4:
  // 36 MB 10.7 ms, 24 MB 10.1 ms, 12 MB 10.2 ms per host apply)
  (void)launches_per_stage;
  int64_t chunk_bytes = 24ll << 20;
  const char* cb = getenv("SIPG_STREAM_CHUNK_BYTES");
  if (cb) chunk_bytes = atoll(cb);
  const int K = make_chunks(p, ndof, chunk_bytes);
  if (K < 2) return false;
  std::vector<int32_t> chunk(nel), stage(nel);
  {
    int k = 0;
    for (int64_t e = 0; e < nel; ++e) {
      while (d->dof_off[e + 1] > p->chunk_dof[k + 1]) ++k;
      chunk[e] = k;
    }
  }
  const H3Slot* sl = (const H3Slot*)d->slots;
  for (int64_t e = 0; e < nel; ++e) {
    int st = chunk[e];
    for (int64_t q = d->slot_off[e]; q < d->slot_off[e + 1]; ++q)
      if (sl[q].kind == 1 && sl[q].partner >= 0) {
        const int nb = sl[sl[q].partner].elem;
        if (chunk[nb] > st) st = chunk[nb];
      }
    stage[e] = st;
  }
  std::vector<int32_t> rows(d->class_desc, d->class_desc + (int64_t)d->n_classes * CD3_WORDS);
  h->st_pub.assign(K, {});
  h->st_comp.assign(K, {});
  p->pub.assign(K, {});      // the standard plans' stage lists stay empty
  p->comp.assign(K, {});
  for (int c = 0; c < d->n_classes; ++c) {   // stages monotone along each class list
    const int32_t* cd = d->class_desc + c * CD3_WORDS;
    const int32_t* el = d->class_elems + cd[CD3_ELEM_OFF];
    for (int i = 1; i < cd[CD3_COUNT]; ++i)
      if (stage[el[i]] < stage[el[i - 1]]) stage[el[i]] = stage[el[i - 1]];
  }
  p->d2h_stage.assign(K, 0);
  {
    int j = 0;
    for (int64_t e = 0; e < nel; ++e) {
      while (d->dof_off[e] >= p->chunk_dof[j + 1]) ++j;
      for (int jj = j; jj < K && p->chunk_dof[jj] < d->dof_off[e + 1]; ++jj)
        if (stage[e] > p->d2h_stage[jj]) p->d2h_stage[jj] = stage[e];
    }
  }
  for (int c = 0; c < d->n_classes; ++c) {
    const int32_t* cd = d->class_desc + c * CD3_WORDS;
    const int n = cd[CD3_COUNT];
    const int32_t* el = d->class_elems + cd[CD3_ELEM_OFF];
    for (int pass = 0; pass < 2; ++pass) {
      const std::vector<int32_t>& key = pass == 0 ? chunk : stage;
      int i0 = 0;
      while (i0 < n) {
        const int k = key[el[i0]];
        int i1 = i0;
        while (i1 < n && key[el[i1]] == k) ++i1;
        for (int j = i1; j < n; ++j)
          if (key[el[j]] <= k) return false;
        const int r = (int)(rows.size() / CD3_WORDS);
        rows.insert(rows.end(), cd, cd + CD3_WORDS);
        rows[(int64_t)r * CD3_WORDS + CD3_COUNT] = i1 - i0;
        rows[(int64_t)r * CD3_WORDS + CD3_ELEM_OFF] += i0;
        const int cap = pass == 0 ? h->cap_pub[c] : h->cap_apply[c];
        const int groups = (i1 - i0 + h->kern[c]->epc - 1) / h->kern[c]->epc;
        const int g = groups < cap ? groups : cap;
        (pass == 0 ? h->st_pub : h->st_comp)[k].push_back({r, g, h->kern[c], cd[CD3_ELEM_OFF] + i0, cd[CD3_ELEM_OFF] + i1});
        i0 = i1;
      }
    }
  }
  if (upload(rows.data(), (int64_t)rows.size(), &h->rows_d)) return false;
  h->hps = h->hp;
  h->hps.cd = h->rows_d;
  if (h->flux) {   // stage-ordered slot records: [mapped by publish stage | identity by compute stage | mapped by compute stage]
    std::vector<H3FluxRec> sr;
    sr.reserve(h->frec_host.size() * 2);
    auto gather = [&](const std::vector<std::vector<H3State::Launch>>& rows_of, bool mapped, std::vector<int64_t>& off) {
      off.assign(K + 1, 0);
      for (int k = 0; k < K; ++k) {
        off[k] = (int64_t)sr.size();
        for (const auto& L : rows_of[k]) {
          const std::vector<int64_t>& cs = mapped ? h->cs_mp : h->cs_id;
          const int64_t base = mapped ? h->n_id : 0;
          sr.insert(sr.end(), h->frec_host.begin() + base + cs[L.pos0], h->frec_host.begin() + base + cs[L.pos1]);
        }
      }
      off[K] = (int64_t)sr.size();
    };
    gather(h->st_pub, true, h->st_mp);
    gather(h->st_comp, false, h->st_fi);
    gather(h->st_comp, true, h->st_fm);
    if (upload(sr.data(), (int64_t)sr.size(), &h->frec_stage_d)) return false;
    h->hps.frec = h->frec_stage_d;
  }
  p->n_chunks = K;
  return true;
}

// RHS lift of hybrid plans: the apply kernels alone, reading a caller-provided
// trace buffer instead of the published one (same layout: slot pub_self offsets, (u, n.grad u)
// per trace point).  With x = 0 and the Dirichlet data as the boundary slots' own traces this is
// exactly the reference's boundary lift (rhs_assemble, sipg.py:707-717).
int sipg_h3_apply_traces(sipg_plan* p, const double* x_dev, const double* traces_dev, double* y_dev, void* stream) {
  if (!p || !p->h3 || !x_dev || !traces_dev || !y_dev) return fail(SIPG_ERR_ARG, "bad argument");
  H3State* h = p->h3;
  // (u hand-over builds) the apply kernels take u from the publish kernels: run those first, publishing into the plan's own
  // trace buffer (scratch here; the caller's traces are what the flux kernels read)
  for (int c = 0; H3C_UHAND && c < p->n_cls; ++c) {
    const int count = h->cd[c * CD3_WORDS + CD3_COUNT];
    if (count == 0 || h->cd[c * CD3_WORDS + CD3_ROLE] == 2) continue;
    const H3Entry* k = h->kern[c];
    k->pub<<<h->grid_pub[c], k->threads, k->smem_pub, (cudaStream_t)stream>>>(h->hp, c, x_dev, y_dev);
    ++p->launches;
  }
  H3Plan hp = h->hp;
  hp.pub = const_cast<double*>(traces_dev);
  for (int c = 0; c < p->n_cls; ++c) {
    const int count = h->cd[c * CD3_WORDS + CD3_COUNT];
    if (count == 0 || h->cd[c * CD3_WORDS + CD3_ROLE] == 2) continue;
    if (h->flux) {
      const int eo = h->cd[c * CD3_WORDS + CD3_ELEM_OFF];
      h3_slot_launch(p, hp, 2, eo, eo + count, (cudaStream_t)stream);
    }
  }
  for (int c = 0; c < p->n_cls; ++c) {
    const int count = h->cd[c * CD3_WORDS + CD3_COUNT];
    if (count == 0 || h->cd[c * CD3_WORDS + CD3_ROLE] == 2) continue;
    const H3Entry* k = h->kern[c];
    k->apply<<<h->grid_apply[c], k->threads, k->smem_apply, (cudaStream_t)stream>>>(hp, c, x_dev, y_dev);
    ++p->launches;
  }
  CK(cudaGetLastError());
  return 0;
}

int64_t sipg_h3_trace_len(const sipg_plan* p) { return p && p->h3 ? p->h3->n_pub : -1; }

int sipg_h3_set_halo(sipg_plan* p, int32_t rank, int32_t nranks, int32_t n_nbr, const int32_t* nbr_rank,
                     const int64_t* send_off, const int64_t* send_cnt, const int64_t* recv_off,
                     const int64_t* recv_cnt) {
  if (!p || !p->h3 || rank < 0 || nranks < 1 || rank >= nranks || n_nbr < 0 ||
      (n_nbr > 0 && (!nbr_rank || !send_off || !send_cnt || !recv_off || !recv_cnt)))
    return fail(SIPG_ERR_ARG, "sipg_h3_set_halo: bad argument");
  H3State* h = p->h3;
  for (int i = 0; i < n_nbr; ++i) {
    if (nbr_rank[i] < 0 || nbr_rank[i] >= nranks || nbr_rank[i] == rank || send_cnt[i] < 0 || recv_cnt[i] < 0 ||
        send_off[i] < 0 || recv_off[i] < 0 || send_off[i] + send_cnt[i] > h->n_pub ||
        recv_off[i] + recv_cnt[i] > h->n_pub)
      return fail(SIPG_ERR_ARG, "sipg_h3_set_halo: neighbour range outside the published-trace buffer");
  }
  h->rank = rank;
  h->nranks = nranks;
  h->nbr.assign(nbr_rank, nbr_rank + n_nbr);
  h->send_off.assign(send_off, send_off + n_nbr);
  h->send_cnt.assign(send_cnt, send_cnt + n_nbr);
  h->recv_off.assign(recv_off, recv_off + n_nbr);
  h->recv_cnt.assign(recv_cnt, recv_cnt + n_nbr);
  // the receive regions are written only by the exchange: zero them once so that an element
  // applied before the first exchange reads defined data
  for (int i = 0; i < n_nbr; ++i)
    if (recv_cnt[i] > 0) CK(cudaMemset(h->pub + recv_off[i], 0, sizeof(double) * recv_cnt[i]));
  return 0;
}

int sipg_nccl_unique_id(void* out128) {
  if (!out128) return fail(SIPG_ERR_ARG, "null argument");
  const NcclApi& a = nccl();
  if (!a.ok) return fail(SIPG_ERR_COMM, a.err);
  ncclUniqueId id;
  NCK(a.getUniqueId(&id));
  memcpy(out128, &id, sizeof(id));
  return 0;
}

int sipg_comm_init(sipg_plan* p, const void* nccl_unique_id, int32_t rank, int32_t nranks) {
  if (!p || !nccl_unique_id || rank < 0 || rank >= nranks) return fail(SIPG_ERR_ARG, "sipg_comm_init: bad argument");
  if (!p->h3) return fail(SIPG_ERR_UNSUPPORTED, "sipg_comm_init: trace-halo exchange is implemented for hybrid plans");
  H3State* h = p->h3;
  if (h->nranks != nranks || h->rank != rank)
    return fail(SIPG_ERR_ARG, "sipg_comm_init: rank / nranks differ from sipg_h3_set_halo");
  const NcclApi& a = nccl();
  if (!a.ok) return fail(SIPG_ERR_COMM, a.err);
  if (h->comm) {
    a.commDestroy(h->comm);
    h->comm = nullptr;
  }
  ncclUniqueId id;
  memcpy(&id, nccl_unique_id, sizeof(id));
  NCK(a.commInitRank(&h->comm, nranks, id, rank));
  if (!h->s_comm) {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    CK(cudaStreamCreateWithPriority(&h->s_comm, cudaStreamNonBlocking, hi));   // exchange ahead of compute
    CK(cudaEventCreateWithFlags(&h->ev_pub1, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&h->ev_comm, cudaEventDisableTiming));
  }
  return 0;
}

int sipg_h3_halo_copy(sipg_plan* dst, const sipg_plan* src, void* stream) {
  if (!dst || !src || !dst->h3 || !src->h3) return fail(SIPG_ERR_ARG, "sipg_h3_halo_copy: bad argument");
  const H3State *d = dst->h3, *s = src->h3;
  for (size_t i = 0; i < d->nbr.size(); ++i) {
    if (d->nbr[i] != s->rank) continue;
    for (size_t j = 0; j < s->nbr.size(); ++j) {
      if (s->nbr[j] != d->rank) continue;
      if (s->send_cnt[j] != d->recv_cnt[i]) return fail(SIPG_ERR_ARG, "sipg_h3_halo_copy: halo sizes differ");
      if (d->recv_cnt[i] > 0)
        CK(cudaMemcpyAsync(d->pub + d->recv_off[i], s->pub + s->send_off[j], sizeof(double) * d->recv_cnt[i],
                           cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
    }
  }
  return 0;
}

int sipg_h3_plan_create(const sipg_h3_desc* d, sipg_plan** out) {
  if (!d || !out) return fail(SIPG_ERR_ARG, "null argument");
  *out = nullptr;
  if (d->abi_version != SIPG_H3_ABI_VERSION) return fail(SIPG_ERR_ARG, "hybrid plan ABI version mismatch");
  if (d->slot_bytes != (int32_t)sizeof(H3Slot) || d->class_words != CD3_WORDS)
    return fail(SIPG_ERR_ARG, "hybrid plan layout mismatch");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return fail(SIPG_ERR_NO_DEVICE, "no CUDA device available (the SIP apply has no CPU fallback)");
  if (d->n_classes <= 0 || d->n_elements <= 0 || !d->class_desc || !d->class_elems || !d->dof_off ||
      !d->elem_geom || !d->slot_off || !d->slots || !d->tables)
    return fail(SIPG_ERR_ARG, "hybrid plan descriptor: missing arrays");
  static const std::vector<H3Entry> table = [] {
    std::vector<H3Entry> v;
    sipg_register_h3(v);
    return v;
  }();
  sipg_plan* p = new sipg_plan();
  memset(p->bufs, 0, sizeof(p->bufs));
  p->h3 = new H3State();
  H3State* h = p->h3;
  p->n_cls = d->n_classes;
  p->n_dofs = d->n_dofs;
  h->cd.assign(d->class_desc, d->class_desc + (int64_t)d->n_classes * CD3_WORDS);
  for (int c = 0; c < d->n_classes; ++c) {
    const int32_t* cd = d->class_desc + c * CD3_WORDS;
    const H3Entry* k = nullptr;
    for (const auto& e : table)
      if (e.shape == cd[CD3_SHAPE] && e.n == cd[CD3_N] && cd[CD3_Q] == e.n + 1) k = &e;
    if (!k) {
      sipg_plan_destroy(p);
      return fail(SIPG_ERR_UNSUPPORTED, "no sm_100a hybrid kernel for shape=" + std::to_string(cd[CD3_SHAPE]) +
                                            " n_modes=" + std::to_string(cd[CD3_N]));
    }
    h->kern.push_back(k);
    // __constant__ 1-D tables (one (shape, n) class per instantiation; role-split classes share them)
    const double* tab = d->tables;
    cudaError_t e = k->upload(tab + cd[CD3_T_D], tab + cd[CD3_T_A], cd[CD3_SHAPE] == 1 ? tab + cd[CD3_T_C] : nullptr,
                              tab + cd[CD3_T_E], tab + cd[CD3_T_ED], tab + cd[CD3_T_PTS], tab + cd[CD3_T_W]);
    if (e != cudaSuccess) {
      sipg_plan_destroy(p);
      return fail(SIPG_ERR_CUDA, std::string("hybrid constant tables: ") + cudaGetErrorString(e));
    }
  }
  int rc = 0;
  int32_t *cd_d, *ce_d;
  int64_t *dof_d, *so_d;
  double *eg_d, *tab_d;
  H3Slot* sl_d;
  if ((rc = upload(d->class_desc, (int64_t)d->n_classes * CD3_WORDS, &cd_d)) ||
      (rc = upload(d->class_elems, d->n_elements, &ce_d)) || (rc = upload(d->dof_off, d->n_elements + 1, &dof_d)) ||
      (rc = upload(d->elem_geom, d->n_elements * H3_EGEO, &eg_d)) ||
      (rc = upload(d->slot_off, d->n_elements + 1, &so_d)) ||
      (rc = upload((const H3Slot*)d->slots, d->n_slots, &sl_d)) || (rc = upload(d->tables, d->n_tables, &tab_d))) {
    sipg_plan_destroy(p);
    return rc;
  }
  void* b[7] = {cd_d, ce_d, dof_d, eg_d, so_d, sl_d, tab_d};
  memcpy(h->bufs, b, sizeof(b));
  h->n_pub = d->n_pub;
  if (d->n_pub > 0) {
    cudaError_t e = cudaMalloc((void**)&h->pub, sizeof(double) * d->n_pub);
    if (e != cudaSuccess) {
      sipg_plan_destroy(p);
      return fail(SIPG_ERR_CUDA, std::string("published-trace buffer: ") + cudaGetErrorString(e));
    }
  }
  {   // own-grid flux buffer: element e's slots from fb_off[e], 2 q^2 doubles each; flux work list
    std::vector<int64_t> fbo((size_t)d->n_elements + 1, 0);
    std::vector<int32_t> qe(d->n_elements, 0);
    std::vector<H3FluxRec> fr((size_t)d->n_slots);
    h->cs_id.assign((size_t)d->n_elements + 1, 0);
    h->cs_mp.assign((size_t)d->n_elements + 1, 0);
    for (int c = 0; c < d->n_classes; ++c) {
      const int32_t* cd = d->class_desc + c * CD3_WORDS;
      for (int i = 0; i < cd[CD3_COUNT]; ++i) qe[d->class_elems[cd[CD3_ELEM_OFF] + i]] = cd[CD3_Q];
    }
    for (int64_t e = 0; e < d->n_elements; ++e)
      fbo[e + 1] = fbo[e] + 2ll * qe[e] * qe[e] * (d->slot_off[e + 1] - d->slot_off[e]);
    const H3Slot* sl = (const H3Slot*)d->slots;
    for (int64_t q = 0; q < d->n_slots; ++q) h->n_id += sl[q].mkind == MAP_ID;
    int64_t ki = 0, km = 0;
    for (int64_t i = 0; i < d->n_elements; ++i) {   // class-list order
      const int32_t e = d->class_elems[i];
      h->cs_id[i] = ki;
      h->cs_mp[i] = km;
      for (int64_t q = d->slot_off[e]; q < d->slot_off[e + 1]; ++q) {
        const H3Slot& s0 = sl[q];
        fr[s0.mkind == MAP_ID ? ki++ : h->n_id + km++] =
            H3FluxRec{s0.pub_self, s0.pub_other, (fbo[e] + 2ll * qe[e] * qe[e] * (q - d->slot_off[e])) * 16 + qe[e],
                      s0.tau, s0.sJ, s0.nt, s0.mkind | (s0.kind << 8), s0.nab, s0.moff, s0.moff2, s0.wtoff};
      }
    }
    h->cs_id[d->n_elements] = ki;
    h->cs_mp[d->n_elements] = km;
    h->frec_host = fr;
    h->flux = true;
    if ((rc = upload(fbo.data(), d->n_elements + 1, &h->fb_off_d)) || (rc = upload(fr.data(), d->n_slots, &h->frec_d))) {
      sipg_plan_destroy(p);
      return rc;
    }
    {   // u hand-over buffer: q^3 doubles per element (offsets even: 16-byte cp.async)
      std::vector<int64_t> ugo((size_t)d->n_elements + 1, 0);
      for (int64_t e = 0; e < d->n_elements; ++e) ugo[e + 1] = ugo[e] + (((int64_t)qe[e] * qe[e] * qe[e] + 1) & ~1ll);
      if ((rc = upload(ugo.data(), d->n_elements + 1, &h->ug_off_d))) {
        sipg_plan_destroy(p);
        return rc;
      }
      std::vector<long long> es((size_t)d->n_elements * 6);
      for (int64_t i = 0; i < d->n_elements; ++i) {
        const int32_t e = d->class_elems[i];
        long long* r = es.data() + 6 * i;
        r[0] = e;
        r[1] = d->slot_off[e + 1] - d->slot_off[e];
        r[2] = d->dof_off[e];
        r[3] = d->slot_off[e];
        r[4] = fbo[e];
        r[5] = ugo[e];
      }
      if ((rc = upload(es.data(), (int64_t)es.size(), &h->escal_d))) {
        sipg_plan_destroy(p);
        return rc;
      }
      cudaError_t e = H3C_UHAND ? cudaMalloc((void**)&h->ug, sizeof(double) * (ugo[d->n_elements] > 0 ? ugo[d->n_elements] : 2))
                                : cudaSuccess;
      if (e != cudaSuccess) {
        sipg_plan_destroy(p);
        return fail(SIPG_ERR_CUDA, std::string("u hand-over buffer: ") + cudaGetErrorString(e));
      }
    }
    if (h->flux && fbo[d->n_elements] > 0) {
      cudaError_t e = cudaMalloc((void**)&h->fb, sizeof(double) * fbo[d->n_elements]);
      if (e != cudaSuccess) {
        sipg_plan_destroy(p);
        return fail(SIPG_ERR_CUDA, std::string("own-grid flux buffer: ") + cudaGetErrorString(e));
      }
    }
  }
  h->hp = H3Plan{cd_d, ce_d, dof_d, eg_d, so_d, sl_d, tab_d, h->pub, d->lambda, h->fb, h->fb_off_d, h->frec_d, h->ug, h->ug_off_d, h->escal_d};
  h->fork_all = getenv("SIPG_H3_FORK") && atoi(getenv("SIPG_H3_FORK")) != 0;
  for (const H3Entry* k : h->kern) {
    cudaError_t e1 = cudaFuncSetAttribute((const void*)k->pub, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)k->smem_pub);
    cudaError_t e2 = cudaFuncSetAttribute((const void*)k->apply, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)k->smem_apply);
    if (e1 != cudaSuccess || e2 != cudaSuccess) {
      sipg_plan_destroy(p);
      return fail(SIPG_ERR_CUDA, "cudaFuncSetAttribute (hybrid kernels)");
    }
  }
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0) {
    sipg_plan_destroy(p);
    return fail(SIPG_ERR_CUDA, "multiprocessor count query failed");
  }
  p->sms = sms;
  p->stream_trace = getenv("SIPG_STREAM_TRACE") != nullptr;
  p->use_graphs = !getenv("SIPG_NO_GRAPH");
  for (int c = 0; c < p->n_cls; ++c) {
    const H3Entry* k = h->kern[c];
    const int count = h->cd[c * CD3_WORDS + CD3_COUNT];
    int occ_p = 1, occ_a = 1;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_p, (const void*)k->pub, k->threads, k->smem_pub) !=
            cudaSuccess ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_a, (const void*)k->apply, k->threads, k->smem_apply) !=
            cudaSuccess ||
        occ_p <= 0 || occ_a <= 0) {
      sipg_plan_destroy(p);
      return fail(SIPG_ERR_CUDA, "occupancy query failed for a hybrid kernel");
    }
    const int groups = (count + k->epc - 1) / k->epc;   // CTAs work on groups of epc elements
    h->grid_pub.push_back(groups < occ_p * sms ? groups : occ_p * sms);
    h->grid_apply.push_back(groups < occ_a * sms ? groups : occ_a * sms);
    h->cap_pub.push_back(occ_p * sms);
    h->cap_apply.push_back(occ_a * sms);
  }
  p->streamed = !getenv("SIPG_NO_STREAM") && build_stream_schedule_h3(p, d);
  std::vector<H3FluxRec>().swap(h->frec_host);
  *out = p;
  return 0;
}

int sipg_apply_role(sipg_plan* p, int32_t role, const double* x_dev, double* y_dev, void* stream) {
  if (!p || !x_dev || !y_dev) return fail(SIPG_ERR_ARG, "null argument");
  cudaStream_t s = (cudaStream_t)stream;
  if (p->h3) return h3_apply(p, role, x_dev, y_dev, s);
  int rc = 0;
  if (p->need_planes) {
    // publish face planes: role 0 (or all) -> every locally owned element; role 1 -> the
    // ghost layer (its coefficients have just arrived); role -1 -> everything
    auto go = [&](int c) {
      const int32_t* cd = p->cd_host.data() + c * CD_WORDS;
      const int count = cd[CD_COUNT], crole = cd[CD_ROLE];
      if (!p->planes_k[c] || count == 0) return false;
      return role < 0 || (role == 0 && crole != 2) || (role == 1 && crole == 2);
    };
    int n = 0, nsmall = 0;
    for (int c = 0; c < p->n_cls; ++c) {
      if (!go(c)) continue;
      ++n;
      nsmall += publish_grid(p->cd_host.data() + c * CD_WORDS, p->cd_host[c * CD_WORDS + CD_COUNT], p->sms) <
                p->sms * 8;
    }
    if ((rc = group_begin(p, s, n, nsmall))) return rc;
    for (int c = 0; c < p->n_cls; ++c) {
      if (!go(c)) continue;
      const int32_t* cd = p->cd_host.data() + c * CD_WORDS;
      p->planes_k[c]->fn<<<publish_grid(cd, cd[CD_COUNT], p->sms), cd[CD_SHAPE] == SHAPE_HEX ? 128 : 256, 0,
                           group_stream(p)>>>(p->dp, c, x_dev);
      ++p->launches;
    }
    if ((rc = group_end(p))) return rc;
  }
  auto go = [&](int c) {
    const int32_t* cd = p->cd_host.data() + c * CD_WORDS;
    return !(cd[CD_COUNT] == 0 || cd[CD_ROLE] == 2 || (role >= 0 && cd[CD_ROLE] != role));
  };
  int n = 0, nsmall = 0;
  for (int c = 0; c < p->n_cls; ++c) {
    if (!go(c)) continue;
    ++n;
    nsmall += p->kern[c]->kind == 0 ? p->grid[c] < p->sms * 8 : p->grid[c] < p->per_sm[c] * p->sms;
  }
  if ((rc = group_begin(p, s, n, nsmall))) return rc;
  for (int c = 0; c < p->n_cls; ++c) {
    if (!go(c)) continue;
    const KernelEntry* k = p->kern[c];
    k->fn<<<p->grid[c], k->threads, k->smem, group_stream(p)>>>(p->dp, c, x_dev, y_dev);
    ++p->launches;
  }
  if ((rc = group_end(p))) return rc;
  CK(cudaGetLastError());
  return 0;
}

// Whole applies are replayed as CUDA graphs: the launch sequence (publishers, element classes, the
// fork / join over side streams) is captured once per (x, y) pair on a private stream and relaunched
// with one cudaGraphLaunch (configs 0 / 1 are launch-latency bound: 6-48 kernels of a few us).
// Distributed plans (an NCCL exchange inside the apply) run eagerly.  SIPG_NO_GRAPH=1 disables it.
int sipg_apply(sipg_plan* p, const double* x_dev, double* y_dev, void* stream) {
  if (!p || !x_dev || !y_dev) return fail(SIPG_ERR_ARG, "null argument");
  const bool dist = p->h3 && p->h3->nranks > 1;
  if (!p->use_graphs || dist) return sipg_apply_role(p, -1, x_dev, y_dev, stream);
  cudaStream_t s = (cudaStream_t)stream;
  for (auto& g : p->graphs)
    if (g.x == x_dev && g.y == y_dev) {
      CK(cudaGraphLaunch(g.exec, s));
      p->launches += g.kernels;
      return 0;
    }
  if (!p->cap_stream) CK(cudaStreamCreateWithFlags(&p->cap_stream, cudaStreamNonBlocking));
  if (int rcf = fork_create(p)) return rcf;   // no resource creation inside the capture
  const int64_t l0 = p->launches;
  CK(cudaStreamBeginCapture(p->cap_stream, cudaStreamCaptureModeThreadLocal));
  int rc = sipg_apply_role(p, -1, x_dev, y_dev, p->cap_stream);
  cudaGraph_t graph = nullptr;
  cudaError_t e = cudaStreamEndCapture(p->cap_stream, &graph);
  if (rc || e != cudaSuccess) {
    if (graph) cudaGraphDestroy(graph);
    cudaGetLastError();
    p->launches = l0;
    if (rc) return rc;
    p->use_graphs = false;      // capture unsupported here: eager from now on
    return sipg_apply_role(p, -1, x_dev, y_dev, stream);
  }
  cudaGraphExec_t exec = nullptr;
  e = cudaGraphInstantiate(&exec, graph, 0);
  cudaGraphDestroy(graph);
  if (e != cudaSuccess) {
    cudaGetLastError();
    p->launches = l0;
    p->use_graphs = false;
    return sipg_apply_role(p, -1, x_dev, y_dev, stream);
  }
  if (p->graphs.size() >= 8) {   // small cache: solvers cycle through a few (x, y) pairs
    cudaGraphExecDestroy(p->graphs.front().exec);
    p->graphs.erase(p->graphs.begin());
  }
  p->graphs.push_back({x_dev, y_dev, exec, p->launches - l0});
  p->launches = l0;
  CK(cudaGraphLaunch(exec, s));
  p->launches += p->graphs.back().kernels;
  return 0;
}

int sipg_apply_class(sipg_plan* p, int32_t cls, const double* x_dev, double* y_dev, void* stream) {
  if (!p || !x_dev || !y_dev || cls < 0 || (cls >= p->n_cls && !p->h3)) return fail(SIPG_ERR_ARG, "bad argument");
  if (p->h3) {   // hybrid plans: launch units 0..n-1 = publish, n..2n-1 = apply, 2n..3n-1 = flux kernels
    if (cls >= 3 * p->n_cls) return fail(SIPG_ERR_ARG, "bad argument");
    H3State* h = p->h3;
    const int c = cls % p->n_cls;
    const int count = h->cd[c * CD3_WORDS + CD3_COUNT];
    const H3Entry* k = h->kern[c];
    if (count == 0 || (cls >= 2 * p->n_cls && !h->flux)) return 0;
    if (cls < p->n_cls) {
      k->pub<<<h->grid_pub[c], k->threads, k->smem_pub, (cudaStream_t)stream>>>(h->hp, c, x_dev, y_dev);
      if (h->flux) {
        const int eo = h->cd[c * CD3_WORDS + CD3_ELEM_OFF];
        h3_slot_launch(p, h->hp, 3, eo, eo + count, (cudaStream_t)stream);
      }
    } else if (cls < 2 * p->n_cls)
      k->apply<<<h->grid_apply[c], k->threads, k->smem_apply, (cudaStream_t)stream>>>(h->hp, c, x_dev, y_dev);
    else {
      const int eo = h->cd[c * CD3_WORDS + CD3_ELEM_OFF];
      h3_slot_launch(p, h->hp, 2, eo, eo + count, (cudaStream_t)stream);
    }
    ++p->launches;
    CK(cudaGetLastError());
    return 0;
  }
  const int count = p->cd_host[cls * CD_WORDS + CD_COUNT];
  if (count == 0) return 0;
  const KernelEntry* k = p->kern[cls];
  k->fn<<<p->grid[cls], k->threads, k->smem, (cudaStream_t)stream>>>(p->dp, cls, x_dev, y_dev);
  ++p->launches;
  CK(cudaGetLastError());
  return 0;
}

int sipg_plan_class_info(const sipg_plan* p, int32_t cls, int32_t* out6) {
  if (!p || cls < 0 || !out6 || cls >= (p->h3 ? 3 : 1) * p->n_cls) return fail(SIPG_ERR_ARG, "bad argument");
  if (p->h3) {   // shape codes 3/4/5 = hex/prism/tet of a hybrid plan; kernel kind 8 publish, 9 apply, 10 flux
    const int32_t* cd = p->h3->cd.data() + (cls % p->n_cls) * CD3_WORDS;
    out6[0] = 3 + cd[CD3_SHAPE]; out6[1] = cd[CD3_N]; out6[2] = cd[CD3_Q]; out6[3] = 0;
    out6[4] = cls >= 2 * p->n_cls && !p->h3->flux ? 0 : cd[CD3_COUNT];
    out6[5] = cls < p->n_cls ? 8 : (cls < 2 * p->n_cls ? 9 : 10);
    return 0;
  }
  const int32_t* cd = p->cd_host.data() + cls * CD_WORDS;
  out6[0] = cd[CD_SHAPE]; out6[1] = cd[CD_N]; out6[2] = cd[CD_Q0]; out6[3] = cd[CD_GEOM]; out6[4] = cd[CD_COUNT];
  out6[5] = p->kern[cls]->kind;
  return 0;
}

static int apply_host_impl(sipg_plan* p, const double* x_host, double* y_host, cudaStream_t s);
static int enqueue_streamed(sipg_plan* p, const double* x_host, double* y_host, cudaStream_t s);

int sipg_apply_host(sipg_plan* p, const double* x_host, double* y_host, void* stream) {
  if (!p || !x_host || !y_host) return fail(SIPG_ERR_ARG, "null argument");
  cudaStream_t s = (cudaStream_t)stream;
  const size_t bytes = sizeof(double) * (size_t)p->n_dofs;
  if (!p->x_stage || !p->y_stage) {   // both staging buffers or neither
    if (p->x_stage) cudaFree(p->x_stage);
    if (p->y_stage) cudaFree(p->y_stage);
    p->x_stage = p->y_stage = nullptr;
    double *xs = nullptr, *ys = nullptr;
    if (cudaMalloc((void**)&xs, bytes) != cudaSuccess || cudaMalloc((void**)&ys, bytes) != cudaSuccess) {
      if (xs) cudaFree(xs);
      cudaGetLastError();
      return fail(SIPG_ERR_CUDA, "host-apply staging buffers: out of device memory");
    }
    p->x_stage = xs;
    p->y_stage = ys;
  }
  const int rc = apply_host_impl(p, x_host, y_host, s);
  if (rc) {
    // copies that target the caller's host buffers may already be queued: drain them before the
    // caller can free or reuse x_host / y_host (their own errors are superseded by rc)
    if (p->s_h2d) cudaStreamSynchronize(p->s_h2d);
    if (p->s_d2h) cudaStreamSynchronize(p->s_d2h);
    cudaStreamSynchronize(s);
  }
  return rc;
}

static int apply_host_impl(sipg_plan* p, const double* x_host, double* y_host, cudaStream_t s) {
  const size_t bytes = sizeof(double) * (size_t)p->n_dofs;
  void* stream = (void*)s;
  if (!p->streamed) {
    CK(cudaMemcpyAsync(p->x_stage, x_host, bytes, cudaMemcpyHostToDevice, s));
    int rc = sipg_apply(p, p->x_stage, p->y_stage, stream);
    if (rc) return rc;
    CK(cudaMemcpyAsync(y_host, p->y_stage, bytes, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return 0;
  }
  const int K = p->n_chunks;
  if (!p->s_h2d) {
    CK(cudaStreamCreateWithFlags(&p->s_h2d, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&p->s_d2h, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&p->ev_start, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&p->ev_done, cudaEventDisableTiming));
    p->ev_h2d.resize(K);
    p->ev_comp.resize(K);
    for (int k = 0; k < K; ++k) {
      CK(cudaEventCreateWithFlags(&p->ev_h2d[k], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&p->ev_comp[k], cudaEventDisableTiming));
    }
  }
  // Replay as a CUDA graph (copies, stage launches and their fork / join captured once per pinned
  // (x_host, y_host) pair): ~400 small launches per host apply on config 4.  Pageable host buffers
  // and the timeline instrumentation run eagerly.
  if (p->use_graphs && !p->stream_trace) {
    cudaPointerAttributes ax{}, ay{};
    const bool pinned = cudaPointerGetAttributes(&ax, x_host) == cudaSuccess &&
                        cudaPointerGetAttributes(&ay, y_host) == cudaSuccess && ax.type == cudaMemoryTypeHost &&
                        ay.type == cudaMemoryTypeHost;
    cudaGetLastError();
    if (pinned) {
      for (auto& g : p->host_graphs)
        if (g.x == x_host && g.y == y_host) {
          CK(cudaGraphLaunch(g.exec, s));
          p->launches += g.kernels;
          CK(cudaStreamSynchronize(s));
          return 0;
        }
      if (!p->cap_stream) CK(cudaStreamCreateWithFlags(&p->cap_stream, cudaStreamNonBlocking));
      if (int rcf = fork_create(p)) return rcf;   // no resource creation inside the capture
      const int64_t l0 = p->launches;
      CK(cudaStreamBeginCapture(p->cap_stream, cudaStreamCaptureModeThreadLocal));
      int rc = enqueue_streamed(p, x_host, y_host, p->cap_stream);
      cudaGraph_t graph = nullptr;
      cudaError_t e = cudaStreamEndCapture(p->cap_stream, &graph);
      cudaGraphExec_t exec = nullptr;
      if (!rc && e == cudaSuccess) e = cudaGraphInstantiate(&exec, graph, 0);
      if (graph) cudaGraphDestroy(graph);
      if (rc) return rc;
      if (e == cudaSuccess) {
        if (p->host_graphs.size() >= 4) {
          cudaGraphExecDestroy(p->host_graphs.front().exec);
          p->host_graphs.erase(p->host_graphs.begin());
        }
        p->host_graphs.push_back({x_host, y_host, exec, p->launches - l0});
        CK(cudaGraphLaunch(exec, s));
        CK(cudaStreamSynchronize(s));
        return 0;
      }
      cudaGetLastError();   // capture unsupported here: eager from now on
      p->launches = l0;
      p->use_graphs = false;
    }
  }
  int rc = enqueue_streamed(p, x_host, y_host, s);
  if (rc) return rc;
  CK(cudaStreamSynchronize(s));
  return 0;
}

// The streamed host apply's work, enqueued on `s` (ends with `s` joined to the copy streams).
static int enqueue_streamed(sipg_plan* p, const double* x_host, double* y_host, cudaStream_t s) {
  const int K = p->n_chunks;
  // SIPG_STREAM_TRACE (instrumentation): timestamps of every chunk copy / stage, printed to stderr
  const bool trace = p->stream_trace;
  static unsigned long long* tbuf = nullptr;
  if (trace && !tbuf) cudaMalloc((void**)&tbuf, sizeof(unsigned long long) * 1024);
  int nmark = 0;
  auto mark = [&](cudaStream_t st) {
    if (!trace || nmark >= 1024) return;
    k_stamp<<<1, 1, 0, st>>>(tbuf, nmark++);
  };
  std::vector<char> tkind;
  // order after whatever the caller queued on `s` (and the previous apply's readers of the stage buffers)
  mark(s); tkind.push_back('S');
  CK(cudaEventRecord(p->ev_start, s));
  CK(cudaStreamWaitEvent(p->s_h2d, p->ev_start, 0));
  CK(cudaStreamWaitEvent(p->s_d2h, p->ev_start, 0));
  for (int k = 0; k < K; ++k) {
    const int64_t a = p->chunk_dof[k], b = p->chunk_dof[k + 1];
    CK(cudaMemcpyAsync(p->x_stage + a, x_host + a, sizeof(double) * (b - a), cudaMemcpyHostToDevice, p->s_h2d));
    CK(cudaEventRecord(p->ev_h2d[k], p->s_h2d));
    mark(p->s_h2d); tkind.push_back('H');
  }
  for (int k = 0; k < K; ++k) {
    CK(cudaStreamWaitEvent(s, p->ev_h2d[k], 0));
#ifdef SIPG_INSTRUMENT
    const bool skip = getenv("SIPG_STREAM_NOCOMPUTE") != nullptr;   // instrumentation build: copies only
#else
    const bool skip = false;
#endif
    if (p->h3 && !skip) {   // each stage's rows are small: run them side by side (fork / join)
      H3State* h = p->h3;
      int rc = group_begin(p, s, (int)h->st_pub[k].size(), (int)h->st_pub[k].size());
      if (rc) return rc;
      for (const auto& L : h->st_pub[k]) {
        cudaStream_t st = group_stream(p);
        L.k->pub<<<L.grid, L.k->threads, L.k->smem_pub, st>>>(h->hps, L.row, p->x_stage, p->y_stage);
        ++p->launches;
      }
      if ((rc = group_end(p))) return rc;
      if (h->flux) {   // the stage's slot kernels, one launch each over its stage-ordered records
        if (h->st_mp[k + 1] > h->st_mp[k]) {
          sipg_h3c_map_launch(h->hps, h->st_mp[k], h->st_mp[k + 1] - h->st_mp[k], p->sms, s);
          ++p->launches;
        }
        if (h->st_fi[k + 1] > h->st_fi[k]) {
          sipg_h3c_flux_launch(h->hps, h->st_fi[k], h->st_fi[k + 1] - h->st_fi[k], false, p->sms, s);
          ++p->launches;
        }
        if (h->st_fm[k + 1] > h->st_fm[k]) {
          sipg_h3c_flux_launch(h->hps, h->st_fm[k], h->st_fm[k + 1] - h->st_fm[k], true, p->sms, s);
          ++p->launches;
        }
      }
      if ((rc = group_begin(p, s, (int)h->st_comp[k].size(), (int)h->st_comp[k].size()))) return rc;
      for (const auto& L : h->st_comp[k]) {
        cudaStream_t st = group_stream(p);
        L.k->apply<<<L.grid, L.k->threads, L.k->smem_apply, st>>>(h->hps, L.row, p->x_stage, p->y_stage);
        ++p->launches;
      }
      if ((rc = group_end(p))) return rc;
    }
    if (!p->h3 && !skip) {   // standard plans: the stage's publishers, then its element rows
      int rc = group_begin(p, s, (int)p->pub[k].size(), (int)p->pub[k].size());
      if (rc) return rc;
      for (const auto& L : p->pub[k]) {
        L.pe->fn<<<L.grid, p->dps.dim == 3 ? 128 : 256, 0, group_stream(p)>>>(p->dps, L.row, p->x_stage);
        ++p->launches;
      }
      if ((rc = group_end(p))) return rc;
      if ((rc = group_begin(p, s, (int)p->comp[k].size(), (int)p->comp[k].size()))) return rc;
      for (const auto& L : p->comp[k]) {
        L.k->fn<<<L.grid, L.k->threads, L.k->smem, group_stream(p)>>>(p->dps, L.row, p->x_stage, p->y_stage);
        ++p->launches;
      }
      if ((rc = group_end(p))) return rc;
    }
    CK(cudaEventRecord(p->ev_comp[k], s));
    mark(s); tkind.push_back('C');
    for (int j = 0; j < K; ++j) {
      if (p->d2h_stage[j] != k) continue;
      const int64_t a = p->chunk_dof[j], b = p->chunk_dof[j + 1];
#ifdef SIPG_INSTRUMENT
      // SIPG_STREAM_DIAG=1 (instrumentation build, wrong results): D2H gated on the copies only
      static const bool diag = getenv("SIPG_STREAM_DIAG") != nullptr;
#else
      const bool diag = false;
#endif
      CK(cudaStreamWaitEvent(p->s_d2h, diag ? p->ev_h2d[k] : p->ev_comp[k], 0));
      CK(cudaMemcpyAsync(y_host + a, p->y_stage + a, sizeof(double) * (b - a), cudaMemcpyDeviceToHost, p->s_d2h));
      mark(p->s_d2h); tkind.push_back('D');
    }
  }
  CK(cudaGetLastError());
  CK(cudaEventRecord(p->ev_done, p->s_d2h));   // join the copy streams back into s
  CK(cudaStreamWaitEvent(s, p->ev_done, 0));
  if (trace) {
    CK(cudaStreamSynchronize(s));
    std::vector<unsigned long long> t(nmark);
    cudaMemcpy(t.data(), tbuf, sizeof(unsigned long long) * nmark, cudaMemcpyDeviceToHost);
    for (int i = 0; i < nmark; ++i) fprintf(stderr, "%c%.3f ", tkind[i], (double)(t[i] - t[0]) * 1e-6);
    fprintf(stderr, "\n");
  }
  return 0;
}

int64_t sipg_plan_launches(const sipg_plan* p) { return p ? p->launches : -1; }

int sipg_plan_kernels_per_apply(const sipg_plan* p) {
  if (!p) return -1;
  int k = 0;
  if (p->h3) {
    for (int c = 0; c < p->n_cls; ++c) {
      const int32_t* cd = p->h3->cd.data() + c * CD3_WORDS;
      if (cd[CD3_COUNT] > 0) k += cd[CD3_ROLE] == 2 ? 1 : 2;
    }
    return k + (p->h3->flux ? 2 : 0);   // + the trace-map and flux kernels (one launch each over every slot)
  }
  for (int c = 0; c < p->n_cls; ++c) {
    if (p->cd_host[c * CD_WORDS + CD_COUNT] > 0 && p->cd_host[c * CD_WORDS + CD_ROLE] != 2) ++k;
    if (p->cd_host[c * CD_WORDS + CD_COUNT] > 0 && p->planes_k.size() > (size_t)c && p->planes_k[c]) ++k;
  }
  return k;
}

int64_t sipg_plan_n_dofs(const sipg_plan* p) { return p ? p->n_dofs : -1; }

int sipg_plan_stream_chunks(const sipg_plan* p) { return p && p->streamed ? p->n_chunks : 0; }

int sipg_plan_host_launches_per_apply(const sipg_plan* p) {
  if (!p) return -1;
  if (!p->streamed) return sipg_plan_kernels_per_apply(p);
  int k = 0;
  if (p->h3) {
    for (int i = 0; i < p->n_chunks; ++i) {
      k += (int)(p->h3->st_pub[i].size() + p->h3->st_comp[i].size()) + (p->h3->flux ? 3 : 0);
    }
    return k;
  }
  for (int i = 0; i < p->n_chunks; ++i) k += (int)(p->pub[i].size() + p->comp[i].size());
  return k;
}

int sipg_plan_destroy(sipg_plan* p) {
  if (!p) return 0;
  for (auto& g : p->graphs) cudaGraphExecDestroy(g.exec);
  for (auto& g : p->host_graphs) cudaGraphExecDestroy(g.exec);
  if (p->cap_stream) cudaStreamDestroy(p->cap_stream);
  for (cudaStream_t st : p->fork.side)
    if (st) cudaStreamDestroy(st);
  for (cudaEvent_t e : p->fork.ev_join)
    if (e) cudaEventDestroy(e);
  if (p->fork.ev_fork) cudaEventDestroy(p->fork.ev_fork);
  if (p->h3) {
    if (p->h3->comm) nccl().commDestroy(p->h3->comm);
    if (p->h3->s_comm) cudaStreamDestroy(p->h3->s_comm);
    if (p->h3->ev_pub1) cudaEventDestroy(p->h3->ev_pub1);
    if (p->h3->ev_comm) cudaEventDestroy(p->h3->ev_comm);
    for (void* b : p->h3->bufs)
      if (b) cudaFree(b);
    if (p->h3->pub) cudaFree(p->h3->pub);
    if (p->h3->fb) cudaFree(p->h3->fb);
    if (p->h3->fb_off_d) cudaFree(p->h3->fb_off_d);
    if (p->h3->frec_d) cudaFree(p->h3->frec_d);
    if (p->h3->frec_stage_d) cudaFree(p->h3->frec_stage_d);
    if (p->h3->ug) cudaFree(p->h3->ug);
    if (p->h3->ug_off_d) cudaFree(p->h3->ug_off_d);
    if (p->h3->escal_d) cudaFree(p->h3->escal_d);
    if (p->h3->rows_d) cudaFree(p->h3->rows_d);
    delete p->h3;
    p->h3 = nullptr;
  }
  for (void* b : p->bufs)
    if (b) cudaFree(b);
  if (p->planes) cudaFree(p->planes);
  if (p->x_stage) cudaFree(p->x_stage);
  if (p->cds_d) cudaFree(p->cds_d);
  if (p->s_h2d) cudaStreamDestroy(p->s_h2d);
  if (p->s_d2h) cudaStreamDestroy(p->s_d2h);
  for (cudaEvent_t e : p->ev_h2d) cudaEventDestroy(e);
  for (cudaEvent_t e : p->ev_comp) cudaEventDestroy(e);
  if (p->ev_start) cudaEventDestroy(p->ev_start);
  if (p->ev_done) cudaEventDestroy(p->ev_done);
  if (p->y_stage) cudaFree(p->y_stage);
  if (p->ws) cudaFree(p->ws);
  if (p->ws_host) cudaFreeHost(p->ws_host);
  delete p;
  return 0;
}

// Internal (sipg_krylov.cu): the plan's cached solver workspace of at least `bytes` device bytes and
// `host_doubles` pinned host doubles.  One solve per plan at a time (like the staging buffers).
int sipg__workspace(sipg_plan* p, size_t bytes, size_t host_doubles, void** dev, double** host) {
  if (!p || !dev || !host) return SIPG_ERR_ARG;
  if (bytes > p->ws_bytes) {
    if (p->ws) cudaFree(p->ws);
    p->ws = nullptr;
    p->ws_bytes = 0;
    if (cudaMalloc(&p->ws, bytes) != cudaSuccess) {
      cudaGetLastError();
      return SIPG_ERR_CUDA;
    }
    p->ws_bytes = bytes;
  }
  if (host_doubles < 64) host_doubles = 64;
  if (host_doubles > p->ws_host_n) {
    if (p->ws_host) cudaFreeHost(p->ws_host);
    p->ws_host = nullptr;
    p->ws_host_n = 0;
    if (cudaMallocHost((void**)&p->ws_host, host_doubles * sizeof(double)) != cudaSuccess) {
      cudaGetLastError();
      return SIPG_ERR_CUDA;
    }
    p->ws_host_n = host_doubles;
  }
  *dev = p->ws;
  *host = p->ws_host;
  return 0;
}

}  // extern "C"
