"""Device binding of one transport problem: padded HBM copies of C and the
marginals plus the libotb context that owns the scratch (CSR, CG vectors,
partial sums).

A ``Session`` is created on first use and cached on the ``OtProblem``
object, so the reference-style free functions (``compute_p(logplan, gamma,
problem, eta)`` ...) do not re-upload C per call.  With a row range (see
``distributed.py``) the session holds only rows [row_begin, row_end) of C
and attaches an NCCL communicator for the length-n all-reduces.

HBM layout: C and every log plan are stored as
(m_loc, ld) float64 row-major with ld = round_up(n, 32), so every row is
256-byte aligned for the 1-D TMA bulk copies of the dense passes.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import _lib
from .core import OtProblem, RowShardCost, _is_torch, host
from .errors import ShapeMismatch

_SESSION_ATTR = "_otb_sessions"
_CTX_POOL: dict = {}      # (device, m, n, row_begin, row_end, ld) -> idle libotb contexts
_POOL_DEPTH = 2


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("paper_2603_07156_b200 needs a CUDA device (sm_100a); there is no CPU path")
    return torch


def round_up(x: int, k: int) -> int:
    return (x + k - 1) // k * k


_SIDE: dict = {}


def _side_stream(dev):
    """One upload stream per device (created once, not per session)."""
    st = _SIDE.get(dev.index)
    if st is None:
        import torch

        st = _SIDE[dev.index] = torch.cuda.Stream(dev)
    return st


class Session:
    """libotb context bound to (problem, eta) on the current CUDA device."""

    def __init__(self, problem: OtProblem, eta: float, row_begin: int = 0, row_end: int | None = None,
                 comm=None, device=None):
        torch = _torch()
        self.torch = torch
        m, n = problem.shape
        self.m, self.n = m, n
        self.row_begin = row_begin
        self.row_end = m if row_end is None else row_end
        self.m_loc = self.row_end - self.row_begin
        self.ld = round_up(n, 32)
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.eta = None
        dev = self.device
        f64 = torch.float64

        cost = problem.cost
        a_h = host(problem.source_marginal)
        b_h = host(problem.target_marginal)
        if a_h.shape[0] != m or b_h.shape[0] != n:
            raise ShapeMismatch("marginal lengths do not match the cost matrix")
        # padded local rows of C (a CUDA cost that already has this layout —
        # e.g. instances.device_cost with ld — is used in place, not copied)
        rows = slice(self.row_begin, self.row_end)
        if isinstance(cost, RowShardCost):
            if (cost.row0, cost.row0 + cost.rows.shape[0]) != (self.row_begin, self.row_end):
                raise ShapeMismatch("RowShardCost rows do not match this rank's row range")
            cost, rows = cost.rows, slice(0, self.m_loc)
            local_rows = True
        else:
            local_rows = self.m_loc == m
        adopt = (_is_torch(cost) and cost.is_cuda and cost.device == dev and cost.dtype == f64
                 and cost.stride() == (self.ld, 1) and local_rows and cost.storage_offset() == 0
                 and cost.untyped_storage().nbytes() >= self.m_loc * self.ld * 8)
        if adopt:
            self.C = torch.as_strided(cost, (self.m_loc, self.ld), (self.ld, 1))
        else:
            self.C = torch.empty((self.m_loc, self.ld), dtype=f64, device=dev)
            if self.ld > n:
                self.C[:, n:].zero_()
        if adopt:
            sq = torch.linalg.vector_norm(self.C).reshape(1) ** 2   # ||C||_F^2 of the local rows
            if comm is not None and comm.world > 1 and self.m_loc < m:
                comm.all_reduce_(sq)
            self.norm_c = float(torch.sqrt(sq))
        elif _is_torch(cost) and not cost.is_cuda and os.environ.get("OTB_C_SIDE", "1") != "0":
            # host C: uploaded on a side stream, so that the caller's next
            # upload (the log plan) shares the PCIe link with it; ||C|| stays on
            # the device (otb_set_cost_norm_sq).  The first library call on
            # this session makes the library stream wait for it (_ready).
            side = _side_stream(dev)
            side.wait_stream(torch.cuda.current_stream(dev))
            self.C.record_stream(side)   # the allocator must not reuse C before the upload ends
            with torch.cuda.stream(side):
                self.C[:, :n].copy_(cost[rows], non_blocking=True)
                sq = torch.linalg.vector_norm(self.C).reshape(1) ** 2   # ||C||_F^2 of the local rows
                if comm is not None and comm.world > 1:
                    comm.all_reduce_(sq)
                self._c_ready = torch.cuda.Event()
                self._c_ready.record(side)
            self._norm_sq = sq
            self.norm_c = None
        elif _is_torch(cost):
            self.C[:, :n].copy_(cost[rows], non_blocking=True)
            sq = torch.linalg.vector_norm(self.C).reshape(1) ** 2   # ||C||_F^2 of the local rows
            if comm is not None and comm.world > 1:
                comm.all_reduce_(sq)
            self.norm_c = float(torch.sqrt(sq))
        else:
            self.C[:, :n].copy_(torch.from_numpy(np.ascontiguousarray(cost[rows])))
            self.norm_c = float(np.linalg.norm(cost))
        # marginals and their logs (numpy on the host: the reference's bits)
        self.a_host, self.b_host = a_h, b_h
        # one upload for the four vectors: [a | b | log a | log b], segments on
        # 256-byte boundaries, b and log b zero-padded like _vec
        ma, nb = round_up(m, 32), round_up(round_up(n, 2) + 16, 32)
        pack = np.zeros(2 * ma + 2 * nb)
        pack[:m] = a_h
        pack[ma:ma + n] = b_h
        pack[ma + nb:ma + nb + m] = np.log(a_h)
        pack[2 * ma + nb:2 * ma + nb + n] = np.log(b_h)
        vecs = torch.from_numpy(pack).to(dev)
        self.a = vecs[:m]
        self.b = vecs[ma:ma + round_up(n, 2) + 16]
        self.log_a = vecs[ma + nb:ma + nb + m]
        self.log_b = vecs[2 * ma + nb:2 * ma + nb + round_up(n, 2) + 16]
        self.norm_a = float(np.linalg.norm(a_h))
        self.norm_b = float(np.linalg.norm(b_h))
        self.default_anchor = int(np.argmax(a_h))             # sparsify.py:25-27
        self.anchor = None
        self.ctx = C.c_void_p()
        self._pool_key = None if comm is not None else (dev.index, m, n, self.row_begin, self.row_end, self.ld)
        pooled = _CTX_POOL.get(self._pool_key) if self._pool_key is not None else None
        if pooled:
            self.ctx = pooled.pop()
            _lib.check(_lib.lib.otb_set_stream(self.ctx, C.c_void_p(self._stream())))
        else:
            with torch.cuda.device(dev):
                _lib.check(_lib.lib.otb_create(C.byref(self.ctx), m, n, self.row_begin, self.row_end, self.ld,
                                               dev.index, C.c_void_p(self._stream())))
        if comm is not None:
            comm.attach(self)
        self.bind(eta)

    # ------------------------------------------------------------------
    def _stream(self) -> int:
        return self.torch.cuda.current_stream(self.device).cuda_stream

    def sync_stream(self):
        _lib.check(_lib.lib.otb_set_stream(self.ctx, C.c_void_p(self._stream())))

    def _vec(self, v, length=None):
        """Device float64 vector padded to an even length (+16)."""
        torch = self.torch
        length = self.n if length is None else length
        out = torch.zeros(round_up(length, 2) + 16, dtype=torch.float64, device=self.device)
        if _is_torch(v):
            out[:length].copy_(v.reshape(-1)[:length])
        else:
            out[:length].copy_(torch.from_numpy(np.ascontiguousarray(np.asarray(v, dtype=np.float64))))
        return out

    def new_vec(self, length=None):
        length = self.n if length is None else length
        return self.torch.zeros(round_up(length, 2) + 16, dtype=self.torch.float64, device=self.device)

    def new_plan(self):
        return self.torch.empty((self.m_loc, self.ld), dtype=self.torch.float64, device=self.device)

    def set_precond(self, kind: str | None):
        """CG preconditioner of this context: None (plain CG) or "jacobi"."""
        code = {None: 0, "jacobi": 1}[kind]
        if getattr(self, "_precond", 0) != code:
            _lib.check(_lib.lib.otb_set_cg_precond(self.ctx, code))
            self._precond = code
            self._last_sparsify = None

    def bind(self, eta: float, anchor: int | None = None):
        eta = float(eta)
        anchor = self.default_anchor if anchor is None else int(anchor)
        if eta == self.eta and anchor == self.anchor:
            return
        _lib.check(_lib.lib.otb_bind(self.ctx, self.C.data_ptr(), self.a.data_ptr(), self.b.data_ptr(),
                                     self.log_a.data_ptr(), self.log_b.data_ptr(), eta, anchor,
                                     0.0 if self.norm_c is None else self.norm_c, self.norm_a, self.norm_b))
        if self.norm_c is None and getattr(self, "_c_ready", None) is None:
            _lib.check(_lib.lib.otb_set_cost_norm_sq(self.ctx, self._norm_sq.data_ptr()))
        self.eta = eta
        self.anchor = anchor

    def _ready(self):
        """Make the current stream wait for the side-stream upload of C."""
        ev = getattr(self, "_c_ready", None)
        if ev is not None:
            cur = self.torch.cuda.current_stream(self.device)
            cur.wait_event(ev)
            self._c_ready = None
            self._norm_sq.record_stream(cur)   # read by the library's copy on this stream
            _lib.check(_lib.lib.otb_set_cost_norm_sq(self.ctx, self._norm_sq.data_ptr()))

    @property
    def ops(self) -> "Ops":
        self._ready()
        return Ops(self)

    def plan(self, logplan):
        """Padded device tensor of the local rows of a LogPlan."""
        t = logplan.device_padded(self.ld, self.device) if logplan.shape[0] == self.m_loc else None
        if t is None:
            raise ShapeMismatch("log plan rows do not match the session's row range")
        return t

    def info(self) -> dict:
        out = (C.c_int64 * 24)()
        _lib.check(_lib.lib.otb_info(self.ctx, out))
        keys = ("nt", "ns", "cl", "colw", "nstage", "ncl", "grid", "hv_mode", "hv_grid", "nnz", "capacity",
                "m_loc", "n", "ld", "nranks", "rank", "hv_groups", "cg_fused", "hv_smem_bytes", "launches",
                "rho_dense", "wc_nq", "wc_win", "wc_ncl")
        return dict(zip(keys, list(out)))

    def launches(self) -> int:
        out = C.c_int64()
        _lib.check(_lib.lib.otb_launch_count(self.ctx, C.byref(out)))
        return int(out.value)

    # ------------------------------------------------------------ profiling
    def prof_enable(self, on: bool = True):
        _lib.check(_lib.lib.otb_prof_enable(self.ctx, 1 if on else 0))

    def prof_read(self, reset: bool = True) -> dict:
        ms = (C.c_double * 16)()
        cnt = (C.c_int64 * 16)()
        by = (C.c_double * 16)()
        _lib.check(_lib.lib.otb_prof_read(self.ctx, ms, cnt, by, 1 if reset else 0))
        names = ("eval", "sparsify", "hess_apply", "cg_vector", "test_a", "test_b", "test_c",
                 "warm_zeta", "warm_gamma", "cg_fused")
        return {nm: dict(ms=ms[k], launches=cnt[k], bytes=by[k]) for k, nm in enumerate(names)}

    def close(self):
        """Return the libotb context to the pool (its scratch — CSR capacity,
        CG vectors, partial rows — is reused by the next session of the same
        shape); contexts with an NCCL communicator are destroyed."""
        if self.ctx:
            pool = _CTX_POOL.setdefault(self._pool_key, []) if self._pool_key is not None else None
            if pool is not None and len(pool) < _POOL_DEPTH:
                if getattr(self, "_precond", 0):
                    _lib.lib.otb_set_cg_precond(self.ctx, 0)   # pooled contexts start plain
                pool.append(self.ctx)
            else:
                _lib.lib.otb_destroy(self.ctx)
            self.ctx = C.c_void_p()

    def __del__(self):  # pragma: no cover - interpreter shutdown order varies
        try:
            self.close()
        except Exception:
            pass


def session_for(problem: OtProblem, eta: float, comm=None) -> Session:
    """Cached Session of (problem, current device); rebinds eta if needed."""
    torch = _torch()
    cache = getattr(problem, _SESSION_ATTR, None)
    if cache is None:
        cache = {}
        object.__setattr__(problem, _SESSION_ATTR, cache)
    key = (torch.cuda.current_device(), None if comm is None else id(comm))
    s = cache.get(key)
    if s is None:
        if comm is None:
            s = Session(problem, eta)
        else:
            r0, r1 = comm.row_range(problem.shape[0])
            s = Session(problem, eta, r0, r1, comm=comm)
        cache[key] = s
    s.bind(eta)
    s.sync_stream()
    return s


# ---------------------------------------------------------------------------
# thin wrappers over the C ABI (device tensors in, scalars out)
# ---------------------------------------------------------------------------

def _ptr(t) -> int:
    return 0 if t is None else t.data_ptr()


class Ops:
    """Entry points of libotb on a Session; every call is stream-ordered on
    torch's current stream and returns host scalars only."""

    def __init__(self, s: Session):
        self.s = s

    def eval(self, plan_t, gamma_t, lse_out=None, grad_out=None):
        out = _lib.EvalOut()
        _lib.check(_lib.lib.otb_eval(self.s.ctx, plan_t.data_ptr(), gamma_t.data_ptr(), _ptr(lse_out),
                                     _ptr(grad_out), C.byref(out)))
        return out.value, out.grad_norm

    def sparsify(self, plan_t, gamma_t, rho: float) -> int:
        nnz = C.c_int64()
        _lib.check(_lib.lib.otb_sparsify(self.s.ctx, plan_t.data_ptr(), gamma_t.data_ptr(), float(rho),
                                         C.byref(nnz)))
        return int(nnz.value)

    def csr_export(self, nnz: int):
        torch = self.s.torch
        dev = self.s.device
        row_ptr = torch.empty(self.s.m_loc + 1, dtype=torch.int64, device=dev)
        cols = torch.empty(max(nnz, 1), dtype=torch.int32, device=dev)
        vals = torch.empty(max(nnz, 1), dtype=torch.float64, device=dev)
        d = self.s.new_vec()
        _lib.check(_lib.lib.otb_csr_export(self.s.ctx, row_ptr.data_ptr(), cols.data_ptr(), vals.data_ptr(),
                                           d.data_ptr()))
        return row_ptr, cols[:nnz], vals[:nnz], d[: self.s.n]

    def hess_apply(self, v_t, shift: float = 0.0, out=None):
        out = self.s.new_vec() if out is None else out
        _lib.check(_lib.lib.otb_hess_apply(self.s.ctx, v_t.data_ptr(), float(shift), out.data_ptr()))
        return out

    def cg(self, shift, rhs_t, rel_tol, max_iters, x_out=None):
        x_out = self.s.new_vec() if x_out is None else x_out
        out = _lib.CgOut()
        _lib.check(_lib.lib.otb_cg(self.s.ctx, float(shift), rhs_t.data_ptr(), float(rel_tol), int(max_iters),
                                   x_out.data_ptr(), C.byref(out)))
        return x_out, int(out.iters), float(out.residual)

    def newton_step(self, plan_t, gamma_in, gamma_out, sigma, beta, cg_rel_tol, cg_max_iters, rho=None):
        p = _lib.NewtonParams(float(sigma), float(beta), float(cg_rel_tol),
                              0 if cg_max_iters is None else int(cg_max_iters),
                              -1.0 if rho is None else float(rho))
        out = _lib.NewtonOut()
        _lib.check(_lib.lib.otb_newton_step(self.s.ctx, plan_t.data_ptr(), gamma_in.data_ptr(),
                                            gamma_out.data_ptr(), C.byref(p), C.byref(out)))
        return out

    def inner_iteration(self, plan_t, gamma_in, gamma_out, sigma, beta, cg_rel_tol, cg_max_iters, eval_first,
                        floor, test_below, out_plan, gamma_src=None):
        """One iteration of inner_solve's loop in native code (otb_inner_iteration):
        [eval], floor stop, Newton step, and the inexact test when the new
        ||g|| < test_below (test_below < 0: never)."""
        p = _lib.NewtonParams(float(sigma), float(beta), float(cg_rel_tol),
                              0 if cg_max_iters is None else int(cg_max_iters), -1.0)
        out = _lib.InnerOut()
        _lib.check(_lib.lib.otb_inner_iteration(self.s.ctx, plan_t.data_ptr(), gamma_in.data_ptr(),
                                                gamma_out.data_ptr(), C.byref(p), 1 if eval_first else 0,
                                                float(floor), float(test_below), _ptr(out_plan), _ptr(gamma_src),
                                                C.byref(out)))
        return out

    def recover_round(self, plan_t, gamma_t, out_plan=None, recover=True, metrics=True):
        res = _lib.TestOut()
        _lib.check(_lib.lib.otb_recover_round(self.s.ctx, plan_t.data_ptr(), gamma_t.data_ptr(), _ptr(out_plan),
                                              1 if recover else 0, 1 if metrics else 0, C.byref(res)))
        return res

    def materialize_rounded(self):
        out = self.s.torch.empty((self.s.m_loc, self.s.n), dtype=self.s.torch.float64, device=self.s.device)
        _lib.check(_lib.lib.otb_materialize_rounded(self.s.ctx, out.data_ptr(), self.s.n))
        return out

    def materialize_p(self, plan_t, gamma_t):
        out = self.s.torch.empty((self.s.m_loc, self.s.n), dtype=self.s.torch.float64, device=self.s.device)
        _lib.check(_lib.lib.otb_materialize_p(self.s.ctx, plan_t.data_ptr(), gamma_t.data_ptr(), out.data_ptr(),
                                              self.s.n))
        return out

    def warm_start(self, plan_t, gamma_t, zeta_t, warm_tol, max_sweeps):
        out = _lib.WarmOut()
        _lib.check(_lib.lib.otb_warm_start(self.s.ctx, plan_t.data_ptr(), gamma_t.data_ptr(), zeta_t.data_ptr(),
                                           float(warm_tol), int(max_sweeps), C.byref(out)))
        return int(out.sweeps), float(out.err)

    def sinkhorn_zeta(self, plan_t, gamma_t, zeta_t) -> float:
        err = C.c_double()
        _lib.check(_lib.lib.otb_sinkhorn_zeta(self.s.ctx, plan_t.data_ptr(), gamma_t.data_ptr(), zeta_t.data_ptr(),
                                              C.byref(err)))
        return float(err.value)

    def sinkhorn_gamma(self, plan_t, gamma_t, zeta_t):
        _lib.check(_lib.lib.otb_sinkhorn_gamma(self.s.ctx, plan_t.data_ptr(), gamma_t.data_ptr(), zeta_t.data_ptr()))

    def scaled_plan(self, plan_t, gamma_t, zeta_t, out_t):
        _lib.check(_lib.lib.otb_scaled_plan(self.s.ctx, plan_t.data_ptr(), gamma_t.data_ptr(), zeta_t.data_ptr(),
                                            out_t.data_ptr()))
        return out_t

    def init_plan(self, plan_t):
        _lib.check(_lib.lib.otb_init_plan(self.s.ctx, plan_t.data_ptr()))
        return plan_t

    def zeta_from_lse(self, zeta_t):
        _lib.check(_lib.lib.otb_zeta_from_lse(self.s.ctx, zeta_t.data_ptr()))
        return zeta_t
