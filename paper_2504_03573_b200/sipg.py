"""The SIP-Helmholtz operator: drop-in for the reference's
`dgsipg.sipg.HelmholtzOperator` hot path (reference sipg.py:219-605).

Same constructor signature and public surface (`n_dofs`, `dof_slice`, `exps`,
`factors`, `certificates`, `timers`, `lhs_eval`, `__call__`, `report`,
`rhs_assemble`, `l2_error`); `lhs_eval` runs
the sm_100a kernels in libsipg.so through the C-ABI.  Inputs may be numpy
arrays (copied host->device->host, like the reference returns a new array) or
CUDA torch tensors (zero-copy, enqueued on the current stream, returns a new
CUDA tensor).  There is no CPU path.

Extra keyword arguments (not in the reference):
  tau_rule     "reference": tau = C max(n-1,1)^2 / h (sipg.py:351-360);
               "baseline":  tau = max(n_L, n_R)^2 / h (BASELINE.json "(P+1)^2/h").
  element_roles  per-element launch role for slab decompositions (0 first,
               1 after the halo exchange, 2 ghost: never computed); see
               distributed.py.
  shared_rule  "patched" (default): Gauss-Legendre shared-trace rule on faces
               touching a non-GLL side (the reference produces NaN there,
               SURVEY.md §8c P2); "reference": higher side's kind.
"""
from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np

from . import _native
from .plan import PlanBuilder
from .polylib import BasisKind

__all__ = ["HelmholtzParams", "HelmholtzOperator"]


@dataclass(frozen=True)
class HelmholtzParams:
    """Reaction coefficient and penalty constant (reference sipg.py:64-74)."""
    lambda_: float = 1.0
    tau_constant: float = 10.0


class HelmholtzOperator:
    """Matrix-free SIPG Helmholtz operator y = (lambda M + L_SIP) x on B200."""

    def __init__(self, mesh, order_map, *, basis_kind=BasisKind.LAGRANGE, rule_kinds=None,
                 params: HelmholtzParams = HelmholtzParams(), strategy: str = "p2p",
                 batch_width: int = 4, face_absorb: str = "auto", force_interp: bool = False,
                 p_geom: int = 1, tau_rule: str = "reference", shared_rule: str = "patched",
                 element_roles=None):
        if strategy not in ("p2p", "p2p_forced", "shared_trace"):
            raise ValueError(f"unknown strategy {strategy!r}")
        if face_absorb not in ("auto", "trace_iproduct"):
            raise ValueError(f"unknown face_absorb {face_absorb!r}")
        if tau_rule not in ("reference", "baseline"):
            raise ValueError(f"unknown tau_rule {tau_rule!r}")
        self.mesh, self.order_map, self.params = mesh, order_map, params
        self.strategy, self.face_absorb, self.force_interp = strategy, face_absorb, force_interp
        self.batch_width = max(1, int(batch_width))   # GPU batches by class; accepted for API parity
        self.p_geom = p_geom
        # reference keys (sipg.py:260); the GPU apply runs the reference's phase 1 (volume + trace
        # publish) and phase 2 (flux + lift) inside one kernel sequence, so "phase1" carries the whole
        # device apply of lhs_eval (copies included) and "phase2" stays 0.0
        self.timers = {"phase1": 0.0, "phase2": 0.0, "total": 0.0, "applies": 0, "setup": 0.0}
        self._exps = self._factors = None
        self._pinned = None
        t0 = time.perf_counter()
        if getattr(mesh, "is_hybrid3d", False):
            self._init_hybrid3d(mesh, order_map, basis_kind, params, tau_rule, t0, element_roles)
            return
        self.plan = PlanBuilder(mesh, order_map, basis_kind=basis_kind, rule_kinds=rule_kinds,
                                lambda_=params.lambda_, tau_constant=params.tau_constant,
                                strategy=strategy, face_absorb=face_absorb, force_interp=force_interp,
                                p_geom=p_geom, tau_rule=tau_rule, shared_rule=shared_rule,
                                element_roles=element_roles).build()
        self.n_dofs = self.plan.n_dofs
        self._dof_off = self.plan.dof_off
        self.certificates = self.plan.certificates
        self.native = _native.NativePlan(self.plan)
        self.timers["setup"] = time.perf_counter() - t0

    def _init_hybrid3d(self, mesh, order_map, basis_kind, params, tau_rule, t0, element_roles=None):
        """Config 4 (hex / prism / tet, mesh3d.HybridMesh3D): every coupling on the shared-trace route
        with the BASELINE penalty (plan3d.py; the reference has no prism / tet)."""
        from .plan3d import Plan3DBuilder
        if getattr(basis_kind, "value", basis_kind) != BasisKind.MODIFIED_MODAL.value:
            raise ValueError("hybrid 3-D meshes use the modified modal basis")
        if tau_rule != "baseline":
            raise ValueError("hybrid 3-D meshes use tau_rule='baseline' (max(n_L, n_R)^2 / h)")
        self.plan = Plan3DBuilder(mesh, order_map, lambda_=params.lambda_, element_roles=element_roles).build()
        self.n_dofs = self.plan.n_dofs
        self._dof_off = self.plan.dof_off
        self.certificates = []
        self.native = _native.NativePlan(self.plan)
        self.timers["setup"] = time.perf_counter() - t0

    def rhs_assemble(self, case, bcs):
        """b = -(v, f) + Dirichlet lift (reference sipg.py:697-718), on the GPU: rhs.py for the
        standard plans, rhs3d.py (lift through the apply kernels) for hybrid 3-D plans."""
        if getattr(self.plan, "is_h3", False):
            from .rhs3d import rhs_assemble
        else:
            from .rhs import rhs_assemble
        return rhs_assemble(self, case, bcs)

    def l2_error(self, x, exact) -> float:
        """sqrt(sum_e int (u_h - u)^2 J) with 2 extra points per direction (reference
        sipg.py:720-741), on the GPU."""
        if getattr(self.plan, "is_h3", False):
            from .rhs3d import l2_error
        else:
            from .rhs import l2_error
        return l2_error(self, x, exact)

    @property
    def exps(self) -> list:
        """Per-element expansion (shared per class, like the reference's lru-cached `expansion`,
        sipg.py:262-265): shape, n_modes, n_coeffs, nq, n_phys, ref_weights, xi_phys, eta_phys."""
        if self._exps is None:
            if getattr(self.plan, "is_h3", False):
                self._exps = [self.plan.ct[c] for c in self.plan.class_of]
            else:
                self._exps = list(self.plan.ct)
        return self._exps

    @property
    def factors(self):
        """GeometricFactors of every element (reference sipg.py:266-267, mesh.py:295-357), built
        lazily on first access (setup data, not used by the device apply)."""
        if self._factors is None:
            from .factors import hybrid_factors, standard_factors
            self._factors = hybrid_factors(self.plan) if getattr(self.plan, "is_h3", False) \
                else standard_factors(self.mesh, self.plan)
        return self._factors

    def dof_slice(self, e: int) -> slice:
        return slice(int(self._dof_off[e]), int(self._dof_off[e + 1]))

    def lhs_eval(self, x):
        """Action of the SIPG operator on a global coefficient vector
        (reference sipg.py:558-602)."""
        t0 = time.perf_counter()
        if _is_cuda_tensor(x):
            import torch
            if x.dtype != torch.float64 or x.shape != (self.n_dofs,):
                raise ValueError(f"expected a float64 vector of length {self.n_dofs}")
            x = x.contiguous()
            y = torch.empty_like(x)
            self.native.apply_device(x.data_ptr(), y.data_ptr(), torch.cuda.current_stream().cuda_stream)
        else:
            x = np.asarray(x, dtype=float)
            if x.shape != (self.n_dofs,):
                raise ValueError(f"expected a vector of length {self.n_dofs}")
            # page-locked staging pair owned by the operator: the chunked H2D / D2H of the streamed
            # host apply run at full PCIe rate only from pinned memory
            if self._pinned is None:
                import torch
                self._pinned = (torch.empty(self.n_dofs, dtype=torch.float64).pin_memory(),
                                torch.empty(self.n_dofs, dtype=torch.float64).pin_memory())
            xp, yp = self._pinned
            np.copyto(xp.numpy(), x)
            self.native.apply_host_ptr(xp.data_ptr(), yp.data_ptr())
            y = yp.numpy().copy()
        dt = time.perf_counter() - t0
        self.timers["phase1"] += dt
        self.timers["total"] += dt
        self.timers["applies"] += 1
        return y

    __call__ = lhs_eval

    def apply_into(self, x_ptr: int, y_ptr: int, stream: int = 0) -> None:
        """Raw device-pointer apply (no allocation), for benchmarks and solvers."""
        self.native.apply_device(x_ptr, y_ptr, stream)

    def report(self) -> str:
        """Certificate report for non-conforming interfaces (reference trace.py:109-130)."""
        lines = ["# interface  left(P,Q)  right(P,Q)  strategy  cond1  cond2  required  actual  symmetric"]
        itf = self.mesh.interfaces
        for iid, (sym, c1, c2, req, act), strat in self.certificates:
            (le, _), (re_, _) = itf[iid].left, itf[iid].right
            nm, nq = self.order_map.n_modes, self.order_map.n_quad
            lines.append("%d  P%dQ%d  P%dQ%d  %s  %s  %s  %d  %d  %s" % (
                iid, nm[le], nq[le], nm[re_], nq[re_], strat, "yes" if c1 else "no",
                "yes" if c2 else "no", req, act, "yes" if sym else "no"))
        return "\n".join(lines) + "\n"


def _is_cuda_tensor(x) -> bool:
    mod = type(x).__module__
    return mod.startswith("torch") and getattr(x, "is_cuda", False)
