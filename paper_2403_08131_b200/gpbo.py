"""Thin ctypes binding of libgpbo.so (include/gpbo.h).  Argument marshalling only.

Every numerical step runs in the library's CUDA kernels; there is no Python or CPU fallback.
Arrays may be numpy arrays (host memory -> GPBO_HOST) or CUDA torch tensors (-> GPBO_DEVICE);
all arrays of one call must live in the same space.  Names follow include/gpbo.h.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# GPBO_LIB selects an alternative in-tree build (A/B kernel experiments); default: the package copy
LIB_PATH = os.environ.get("GPBO_LIB") or os.path.join(_HERE, "libgpbo.so")

OK, EINVAL, ENOTPD, WDEGENERATE, ESAMPLING, ECUDA, ENCCL, ENOMEM, ENOTSUP = range(9)
RBF, MATERN52 = 0, 1
HOST, DEVICE = 0, 1
STATUS_NAMES = ["OK", "EINVAL", "ENOTPD", "WDEGENERATE", "ESAMPLING", "ECUDA", "ENCCL",
                "ENOMEM", "ENOTSUP"]
NCCL_ID_BYTES = 128


class GpboError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS_NAMES[status] if 0 <= status < 9 else status}: {msg}")
        self.status = status


class SpaceDesc(C.Structure):
    _fields_ = [("P", C.c_int32), ("kind", C.c_void_p), ("nvals", C.c_void_p), ("lo", C.c_void_p),
                ("hi", C.c_void_p), ("val_off", C.c_void_p), ("values", C.c_void_p),
                ("nblocks", C.c_int32), ("block_off", C.c_void_p), ("block_params", C.c_void_p),
                ("tuple_off", C.c_void_p), ("tuples", C.c_void_p)]


class Ml2Opts(C.Structure):
    _fields_ = [("starts", C.c_int32), ("iters", C.c_int32), ("seed", C.c_uint64),
                ("step", C.c_double), ("ls_lo", C.c_double), ("ls_hi", C.c_double),
                ("sf2_lo", C.c_double), ("sf2_hi", C.c_double), ("sn2_lo", C.c_double),
                ("sn2_hi", C.c_double)]


class PlanArgs(C.Structure):
    _fields_ = [("R", C.c_int32), ("P", C.c_int32), ("parent", C.c_void_p),
                ("has_metric", C.c_void_p), ("owner_off", C.c_void_p), ("owners", C.c_void_p),
                ("shared", C.c_void_p), ("matrix", C.c_void_p), ("cutoff", C.c_double),
                ("dim_cap", C.c_int32), ("budget_mult", C.c_int32), ("budget_floor", C.c_int32)]


class PlanOut(C.Structure):
    _fields_ = [("nsearch", C.c_int32), ("search_stage", C.c_void_p),
                ("search_target", C.c_void_p), ("search_budget", C.c_void_p),
                ("search_dims", C.c_void_p), ("tuned", C.c_void_p), ("dropped", C.c_void_p)]


class FitArgs(C.Structure):
    _fields_ = [("S", C.c_int32), ("n", C.c_void_p), ("d", C.c_void_p), ("X", C.c_void_p),
                ("y", C.c_void_p), ("lengthscale", C.c_void_p), ("signal_var", C.c_void_p),
                ("noise_var", C.c_void_p), ("kernel", C.c_int), ("mem", C.c_int)]


_lib = None


def load():
    """Load the in-tree libgpbo.so; fails loudly when it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with "
                          "`python -c 'import __graft_entry__ as g; g.build()'`")
    lib = C.CDLL(LIB_PATH)
    vp, i32, i64 = C.c_void_p, C.c_int32, C.c_int64
    sig = {
        "gpbo_nccl_unique_id": (C.c_int, [vp]),
        "gpbo_ctx_create": (C.c_int, [C.c_int, vp, C.c_int, C.c_int, vp, C.POINTER(vp)]),
        "gpbo_ctx_destroy": (C.c_int, [vp]),
        "gpbo_last_error": (C.c_char_p, [vp]),
        "gpbo_version": (C.c_char_p, []),
        "gp_fit": (C.c_int, [vp, C.POINTER(FitArgs), C.POINTER(vp), vp, vp]),
        "gp_fit_async": (C.c_int, [vp, C.POINTER(FitArgs), C.POINTER(vp)]),
        "gp_model_sync": (C.c_int, [vp, vp, vp, vp]),
        "gp_model_free": (None, [vp]),
        "gp_model_lml": (C.c_int, [vp, vp]),
        "gp_fit_append": (C.c_int, [vp, vp, vp, vp, C.c_int, C.POINTER(vp), vp, vp]),
        "gpbo_last_append_refit": (i64, [vp]),
        "gp_fit_ml2": (C.c_int, [vp, C.POINTER(FitArgs), C.POINTER(Ml2Opts), vp, vp, vp, vp, vp]),
        "gpbo_last_ml2_evals": (i64, [vp]),
        "gpbo_influence": (C.c_int, [i32, i32, i32, vp, vp, vp, vp]),
        "gpbo_plan": (C.c_int, [C.POINTER(PlanArgs), C.POINTER(PlanOut)]),
        "gpbo_nm_selftest": (C.c_int, [C.c_int, vp, vp, vp, C.c_double, C.c_int, vp, vp, vp, vp,
                                       vp, vp]),
        "gp_model_stats": (C.c_int, [vp, i32, vp, vp, vp, vp]),
        "gp_model_export": (C.c_int, [vp, vp, i32, vp, vp, vp]),
        "gp_posterior": (C.c_int, [vp, vp, i32, vp, i64, C.c_int, vp, vp, vp]),
        "ei_score_argmax": (C.c_int, [vp, vp, vp, vp, vp, vp, C.c_int, vp, vp]),
        "gpbo_launch_count": (i64, [vp]),
        "gpbo_last_refine_count": (i64, [vp]),
        "gpbo_collective_count": (i64, [vp]),
        "gpbo_last_bracket_violations": (i64, [vp]),
        "gpbo_debug_bound_scale": (C.c_int, [vp, C.c_float]),
        "gpbo_last_score_impl": (C.c_int, [vp]),
        "gpbo_last_tc_pair": (C.c_int, [vp]),
        "gpbo_set_profiling": (C.c_int, [vp, C.c_int]),
        "gpbo_kernel_time": (C.c_int, [vp, C.c_int, vp, vp]),
        "gpbo_set_score_impl": (C.c_int, [vp, C.c_int]),
        "gpbo_debug_fast_phase": (C.c_int, [vp, vp, i32, vp, i64] + [vp] * 6),
        "gpbo_debug_trace": (C.c_int, [vp, vp]),
        "gpbo_tc_bench": (C.c_int, [vp, vp, vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, vp]),
        "gpbo_tc_selftest": (C.c_int, [vp, vp, vp, C.c_int, C.c_int, C.c_int, C.c_int]),
        "gpbo_space_create": (C.c_int, [vp, C.POINTER(SpaceDesc), C.POINTER(vp)]),
        "gpbo_space_free": (None, [vp]),
        "gpbo_space_dim": (i32, [vp]),
        "gpbo_space_encode": (C.c_int, [vp, vp, vp]),
        "gpbo_space_sample": (C.c_int, [vp, vp, C.c_uint64, i32, i32, i64, i64, C.c_int, vp]),
        "bo_suggest_batch": (C.c_int, [vp, vp, vp, vp, C.c_uint64, i32, i32, vp, vp, vp]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


def exported_symbols():
    """Names of the entry points include/gpbo.h declares (for the load/export test)."""
    return ["gpbo_nccl_unique_id", "gpbo_ctx_create", "gpbo_ctx_destroy", "gpbo_last_error",
            "gpbo_version", "gp_fit", "gp_fit_async", "gp_model_sync", "gp_model_free", "gp_model_lml", "gp_fit_append", "gpbo_last_append_refit", "gp_fit_ml2", "gpbo_last_ml2_evals", "gpbo_nm_selftest", "gpbo_influence", "gpbo_plan", "gp_model_stats", "gp_model_export",
            "gp_posterior", "ei_score_argmax", "gpbo_launch_count", "gpbo_collective_count", "gpbo_last_bracket_violations",
            "gpbo_debug_bound_scale", "gpbo_set_score_impl", "gpbo_last_refine_count", "gpbo_last_score_impl",
            "gpbo_last_tc_pair", "gpbo_set_profiling", "gpbo_kernel_time",
            "gpbo_debug_fast_phase", "gpbo_tc_selftest", "gpbo_debug_trace",
            "gpbo_tc_bench", "gpbo_space_create", "gpbo_space_free", "gpbo_space_dim",
            "gpbo_space_encode", "gpbo_space_sample", "bo_suggest_batch"]


def _is_torch(a):
    return type(a).__module__.startswith("torch")


def _ptr(a, dtype):
    """(address, mem) of a contiguous array of the given numpy dtype; None -> (None, None)."""
    if a is None:
        return None, None
    if _is_torch(a):
        import torch
        want = {np.float32: torch.float32, np.float64: torch.float64,
                np.int64: torch.int64, np.int32: torch.int32}[dtype]
        if a.dtype != want or not a.is_contiguous():
            raise TypeError(f"tensor must be contiguous {want}")
        return a.data_ptr(), (DEVICE if a.is_cuda else HOST)
    if not (isinstance(a, np.ndarray) and a.dtype == dtype and a.flags.c_contiguous):
        raise TypeError(f"array must be a C-contiguous numpy {np.dtype(dtype)}")
    return a.ctypes.data, HOST


def _mem_of(*pairs):
    mems = {m for _, m in pairs if m is not None}
    if len(mems) > 1:
        raise TypeError("all arrays of one call must be host or all device")
    return mems.pop() if mems else HOST


class Model:
    def __init__(self, ctx, handle, S, n, d, status, jitter_k):
        self.ctx, self.handle, self.S = ctx, handle, S
        self.n, self.d = list(n), list(d)
        self._status, self._jitter_k = status, jitter_k
        self._inputs = None

    def sync(self):
        """gp_model_sync: fetch the per-search statuses of an asynchronous fit."""
        if self._status is None:
            st = np.zeros(self.S, np.int32)
            jk = np.zeros(self.S, np.int32)
            load().gp_model_sync(self.ctx.handle, self.handle, st.ctypes.data, jk.ctypes.data)
            self._status, self._jitter_k = st, jk
        return self

    @property
    def status(self):
        return self.sync()._status

    @property
    def jitter_k(self):
        return self.sync()._jitter_k

    def stats(self, s):
        lib = load()
        vals = [C.c_double() for _ in range(4)]
        _check(self.ctx, lib.gp_model_stats(self.handle, s, *[C.byref(v) for v in vals]))
        return dict(zip(("mean", "std", "best", "alpha_l1"), (v.value for v in vals)))

    def lml(self):
        """gp_model_lml: log marginal likelihood per search (float64 [S])."""
        out = np.zeros(self.S)
        _check(self.ctx, load().gp_model_lml(self.handle, out.ctypes.data))
        return out

    def export(self, s):
        """float64 (L, L^-1, alpha) of search s (row-major lower triangles)."""
        n = self.n[s]
        L = np.zeros((n, n))
        Li = np.zeros((n, n))
        a = np.zeros(n)
        _check(self.ctx, load().gp_model_export(self.ctx.handle, self.handle, s, L.ctypes.data,
                                                Li.ctypes.data, a.ctypes.data))
        return L, Li, a

    def free(self):
        if self.handle:
            load().gp_model_free(self.handle)
            self.handle = None
        self._inputs = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def _check(ctx, st, ok=(OK,)):
    if st not in ok:
        msg = load().gpbo_last_error(ctx.handle if ctx is not None else None)
        raise GpboError(st, msg.decode() if msg else "")
    return st


def nccl_unique_id():
    buf = (C.c_char * NCCL_ID_BYTES)()
    st = load().gpbo_nccl_unique_id(C.addressof(buf))
    if st != OK:
        raise GpboError(st, "ncclGetUniqueId failed")
    return bytes(buf)


class Context:
    """gpbo_ctx: one per (rank, device, stream)."""

    def __init__(self, device=0, stream=None, nranks=1, rank=0, nccl_id=None):
        lib = load()
        h = C.c_void_p()
        sp = None
        if stream is not None:
            sp = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
        idbuf = None
        if nccl_id is not None:
            idbuf = (C.c_char * NCCL_ID_BYTES).from_buffer_copy(nccl_id)
        st = lib.gpbo_ctx_create(device, sp, nranks, rank,
                                 C.addressof(idbuf) if idbuf is not None else None, C.byref(h))
        if st != OK:
            raise GpboError(st, "gpbo_ctx_create failed")
        self.handle = h
        self.device, self.nranks, self.rank = device, nranks, rank

    def close(self):
        if self.handle:
            load().gpbo_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def launches(self):
        return int(load().gpbo_launch_count(self.handle))

    @property
    def collectives(self):
        """ncclAllReduce calls issued on this ctx's communicator (H10)."""
        return int(load().gpbo_collective_count(self.handle))

    @property
    def last_violations(self):
        """Bracket violations found by the last argmax call (searches re-scored exactly)."""
        return int(load().gpbo_last_bracket_violations(self.handle))

    def debug_bound_scale(self, scale):
        """Test hook: multiply the fast phase's error bounds by `scale`."""
        _check(self, load().gpbo_debug_bound_scale(self.handle, float(scale)))

    @property
    def last_refine_count(self):
        return int(load().gpbo_last_refine_count(self.handle))

    @property
    def last_impl(self):
        return int(load().gpbo_last_score_impl(self.handle))

    @property
    def last_tc_pair(self):
        return int(load().gpbo_last_tc_pair(self.handle))

    def debug_trace(self, buf):
        """buf: CUDA int64 tensor of >= 65536 entries, or None to disable."""
        _check(self, load().gpbo_debug_trace(self.handle, None if buf is None else buf.data_ptr()))

    def set_profiling(self, on=True):
        _check(self, load().gpbo_set_profiling(self.handle, int(bool(on))))

    KERNELS = ("fit", "fast", "refine", "pack", "mean")

    def kernel_time(self, kind):
        """(launches, total ms) of one library kernel kind since set_profiling(True)."""
        k = self.KERNELS.index(kind) if isinstance(kind, str) else int(kind)
        cnt, ms = C.c_int64(), C.c_double()
        _check(self, load().gpbo_kernel_time(self.handle, k, C.byref(cnt), C.byref(ms)))
        return cnt.value, ms.value

    def set_score_impl(self, impl):
        """0 auto, 1 CUDA-core, 2 tcgen05 (see include/gpbo.h)."""
        _check(self, load().gpbo_set_score_impl(self.handle, int(impl)))

    def fit(self, n, d, X, y, lengthscale, signal_var, noise_var, kernel=MATERN52, wait=True):
        """gp_fit over a ragged batch; returns a Model (status per search in model.status).
        wait=False: gp_fit_async (statuses fetched on first access of model.status)."""
        lib = load()
        S = len(n)
        n_a = np.ascontiguousarray(n, dtype=np.int32)
        d_a = np.ascontiguousarray(d, dtype=np.int32)
        ptrs = [_ptr(X, np.float32), _ptr(y, np.float64), _ptr(lengthscale, np.float32),
                _ptr(signal_var, np.float32), _ptr(noise_var, np.float32)]
        mem = _mem_of(*ptrs)
        args = FitArgs(S, n_a.ctypes.data, d_a.ctypes.data, ptrs[0][0], ptrs[1][0], ptrs[2][0],
                       ptrs[3][0], ptrs[4][0], int(kernel), mem)
        h = C.c_void_p()
        if not wait:
            _check(self, lib.gp_fit_async(self.handle, C.byref(args), C.byref(h)))
            m = Model(self, h, S, n_a, d_a, None, None)
            # the kernels read the inputs asynchronously (include/gpbo.h, gp_fit_async lifetime)
            m._inputs = (X, y, lengthscale, signal_var, noise_var)
            return m
        status = np.zeros(S, np.int32)
        jk = np.zeros(S, np.int32)
        st = lib.gp_fit(self.handle, C.byref(args), C.byref(h), status.ctypes.data,
                        jk.ctypes.data)
        _check(self, st, ok=(OK, ENOTPD, WDEGENERATE))
        return Model(self, h, S, n_a, d_a, status, jk)

    def fit_append(self, model, x_new, y_new):
        """gp_fit_append: model + one new observation per search (x_new [sum d], y_new [S]) ->
        a new Model (O(n^2) bordered update; the previous model is unchanged)."""
        px, m1 = _ptr(x_new, np.float32)
        py, m2 = _ptr(y_new, np.float64)
        mem = _mem_of((px, m1), (py, m2))
        S = model.S
        h = C.c_void_p()
        status = np.zeros(S, np.int32)
        jk = np.zeros(S, np.int32)
        st = load().gp_fit_append(self.handle, model.handle, px, py, mem, C.byref(h),
                                  status.ctypes.data, jk.ctypes.data)
        _check(self, st, ok=(OK, ENOTPD, WDEGENERATE))
        m = Model(self, h, S, [n + 1 for n in model.n], model.d, status, jk)
        m._inputs = (x_new, y_new)
        return m

    @property
    def last_append_refit(self):
        return int(load().gpbo_last_append_refit(self.handle))

    def fit_ml2(self, n, d, X, y, lengthscale, signal_var, noise_var, kernel=MATERN52,
                starts=8, iters=200, seed=0, step=0.5, bounds=((1e-3, 10.0), (1e-3, 1e3),
                                                               (1e-6, 1.0))):
        """gp_fit_ml2 (host numpy inputs; theta = start 0) -> dict(ls, sf2, sn2, lml,
        lml_starts [S, starts], evals)."""
        S = len(n)
        n_a = np.ascontiguousarray(n, dtype=np.int32)
        d_a = np.ascontiguousarray(d, dtype=np.int32)
        arrs = [np.ascontiguousarray(X, np.float32), np.ascontiguousarray(y, np.float64),
                np.ascontiguousarray(lengthscale, np.float32),
                np.ascontiguousarray(signal_var, np.float32),
                np.ascontiguousarray(noise_var, np.float32)]
        args = FitArgs(S, n_a.ctypes.data, d_a.ctypes.data, *[a.ctypes.data for a in arrs],
                       int(kernel), HOST)
        (l0, l1), (f0, f1), (s0, s1) = bounds
        opts = Ml2Opts(int(starts), int(iters), int(seed), float(step), l0, l1, f0, f1, s0, s1)
        ls = np.zeros(int(d_a.sum()), np.float32)
        sf2 = np.zeros(S, np.float32)
        sn2 = np.zeros(S, np.float32)
        lml = np.zeros(S)
        lst = np.zeros((S, int(starts)))
        _check(self, load().gp_fit_ml2(self.handle, C.byref(args), C.byref(opts), ls.ctypes.data,
                                       sf2.ctypes.data, sn2.ctypes.data, lml.ctypes.data,
                                       lst.ctypes.data))
        return dict(ls=ls, sf2=sf2, sn2=sn2, lml=lml, lml_starts=lst,
                    evals=int(load().gpbo_last_ml2_evals(self.handle)))

    def posterior(self, model, s, Xstar, want=("mu", "var", "ei")):
        """gp_posterior: raw-unit (mu, var, ei) for every row of X* (same space as X*)."""
        px, mem = _ptr(Xstar, np.float32)
        M = int(Xstar.shape[0])
        outs = []
        for name in ("mu", "var", "ei"):
            if name not in want:
                outs.append(None)
            elif _is_torch(Xstar):
                import torch
                outs.append(torch.empty(M, dtype=torch.float32, device=Xstar.device))
            else:
                outs.append(np.empty(M, np.float32))
        op = [(_ptr(o, np.float32)[0] if o is not None else None) for o in outs]
        _check(self, load().gp_posterior(self.handle, model.handle, s, px, M, mem, *op))
        return tuple(outs)

    def debug_fast_phase(self, model, s, Xstar):
        """Fast-phase values of every candidate (CUDA tensor X*): dict of CUDA tensors
        mu, dmu, var, dvar, ei_lo, ei_hi (standardised units)."""
        import torch
        px, mem = _ptr(Xstar, np.float32)
        if mem != DEVICE:
            raise TypeError("debug_fast_phase needs a CUDA tensor")
        M = int(Xstar.shape[0])
        names = ("mu", "dmu", "var", "dvar", "ei_lo", "ei_hi")
        outs = {k: torch.empty(M, dtype=torch.float32, device=Xstar.device) for k in names}
        _check(self, load().gpbo_debug_fast_phase(self.handle, model.handle, s, px, M,
                                                  *[outs[k].data_ptr() for k in names]))
        return outs

    def score_argmax(self, model, Xstar, m_off, m_global_base=None, best=None):
        """ei_score_argmax -> (idx int64[S], ei float32[S] raw units)."""
        px, mem = _ptr(Xstar, np.float32)
        off = np.ascontiguousarray(m_off, dtype=np.int64)
        base = None if m_global_base is None else np.ascontiguousarray(m_global_base, np.int64)
        b = None if best is None else np.ascontiguousarray(best, np.float64)
        idx = np.zeros(model.S, np.int64)
        ei = np.zeros(model.S, np.float32)
        _check(self, load().ei_score_argmax(
            self.handle, model.handle, px, off.ctypes.data,
            base.ctypes.data if base is not None else None,
            b.ctypes.data if b is not None else None, mem, idx.ctypes.data, ei.ctypes.data))
        return idx, ei


def influence(baseline, variations, valid=None):
    """gpbo_influence (host-only): baseline [R], variations [P, V, R] (routine runtimes),
    valid [P, V] bool or None -> variability matrix [R, P]."""
    b = np.ascontiguousarray(baseline, np.float64)
    v = np.ascontiguousarray(variations, np.float64)
    P, V, R = v.shape
    ok = None if valid is None else np.ascontiguousarray(valid, np.uint8)
    out = np.zeros((R, P))
    st = load().gpbo_influence(R, P, V, b.ctypes.data, v.ctypes.data,
                               ok.ctypes.data if ok is not None else None, out.ctypes.data)
    if st != OK:
        raise GpboError(st, "gpbo_influence: bad arguments (zero baseline?)")
    return out


def plan(matrix, owners, parent=None, has_metric=None, shared=None, cutoff=0.25, dim_cap=10,
         budget_mult=10, budget_floor=10):
    """gpbo_plan (host-only): matrix [R, P]; owners: list (per parameter) of owning routine
    indices -> list of dicts (stage, target, budget, params) and the dropped parameter list."""
    M = np.ascontiguousarray(matrix, np.float64)
    R, P = M.shape
    par = np.ascontiguousarray(parent if parent is not None else [-1] * R, np.int32)
    hm = np.ascontiguousarray(has_metric if has_metric is not None else [1] * R, np.int32)
    off = np.zeros(P + 1, np.int32)
    off[1:] = np.cumsum([len(o) for o in owners])
    own = np.ascontiguousarray([r for o in owners for r in o] + [0], np.int32)
    sh = np.ascontiguousarray(shared if shared is not None else [1] * P, np.int32)
    args = PlanArgs(R, P, par.ctypes.data, hm.ctypes.data, off.ctypes.data, own.ctypes.data,
                    sh.ctypes.data, M.ctypes.data, float(cutoff), int(dim_cap), int(budget_mult),
                    int(budget_floor))
    arr = [np.zeros(R, np.int32) for _ in range(4)]
    tuned = np.zeros((R, P), np.uint8)
    dropped = np.zeros(P, np.uint8)
    out = PlanOut(0, *[a.ctypes.data for a in arr], tuned.ctypes.data, dropped.ctypes.data)
    st = load().gpbo_plan(C.byref(args), C.byref(out))
    if st != OK:
        raise GpboError(st, "gpbo_plan: bad arguments")
    searches = [dict(stage=int(arr[0][s]), target=int(arr[1][s]), budget=int(arr[2][s]),
                     params=[int(p) for p in np.flatnonzero(tuned[s])])
                for s in range(out.nsearch)]
    return searches, [int(p) for p in np.flatnonzero(dropped)]


NM_OBJ = C.CFUNCTYPE(C.c_double, C.POINTER(C.c_double), C.c_void_p)


def nm_selftest(f, x0, lo, hi, step=0.5, iters=200):
    """Host-only: the library's Nelder-Mead on a Python objective f(x) -> (x, f, f0, nevals)."""
    x0 = np.ascontiguousarray(x0, np.float64)
    lo = np.ascontiguousarray(lo, np.float64)
    hi = np.ascontiguousarray(hi, np.float64)
    dim = x0.size
    cb = NM_OBJ(lambda p, u: float(f(np.ctypeslib.as_array(p, shape=(dim,)).copy())))
    bx = np.zeros(dim)
    bf, sf, ne = C.c_double(), C.c_double(), C.c_int64()
    st = load().gpbo_nm_selftest(dim, x0.ctypes.data, lo.ctypes.data, hi.ctypes.data, step, iters,
                                 C.cast(cb, C.c_void_p), None, bx.ctypes.data, C.byref(bf),
                                 C.byref(sf), C.byref(ne))
    if st != OK:
        raise GpboError(st, "nm_selftest failed")
    return bx, bf.value, sf.value, ne.value


def tc_selftest(A, B, row_bytes, b_row_off=0):
    """D = A B^T through the tcgen05 path (A: 128 x K, B: N x K fp16 CUDA tensors)."""
    import torch
    N, K = B.shape
    D = torch.empty(128, N, dtype=torch.float32, device=A.device)
    st = load().gpbo_tc_selftest(A.data_ptr(), B.data_ptr(), D.data_ptr(), N, K, row_bytes,
                                 b_row_off)
    if st != OK:
        raise GpboError(st, "tc_selftest failed")
    return D


class Space:
    """gpbo_space from a parameter list (dicts with kind REAL/INT {lo, hi}, ORDINAL {values},
    CATEGORICAL {K}, FIXED {lo}: a constant, no encoded column) and constrained blocks
    ({params: [...], tuples: [[value indices]...]})."""

    def __init__(self, ctx, params, blocks=()):
        P = len(params)
        kind = np.array([p["kind"] for p in params], np.int32)
        nv = np.array([len(p["values"]) if p["kind"] == 2 else p.get("K", 0) for p in params],
                      np.int32)
        lo = np.array([float(p.get("lo", 0.0)) for p in params])
        hi = np.array([float(p.get("hi", 1.0)) for p in params])
        vals, voff = [], []
        for p in params:
            voff.append(len(vals))
            if p["kind"] == 2:
                vals.extend(float(v) for v in p["values"])
        voff = np.array(voff, np.int32)
        vals = np.array(vals + [0.0])
        boff, bpar, toff, tup = [0], [], [0], []
        for b in blocks:
            bpar.extend(b["params"])
            boff.append(len(bpar))
            t = np.asarray(b["tuples"], np.int32).reshape(len(b["tuples"]), len(b["params"]))
            tup.extend(t.ravel().tolist())
            toff.append(toff[-1] + t.shape[0])
        self._keep = [kind, nv, lo, hi, voff, vals] + [np.array(x + [0], np.int32)
                                                       for x in (boff, bpar, toff, tup)]
        k = self._keep
        desc = SpaceDesc(P, k[0].ctypes.data, k[1].ctypes.data, k[2].ctypes.data,
                         k[3].ctypes.data, k[4].ctypes.data, k[5].ctypes.data, len(blocks),
                         k[6].ctypes.data, k[7].ctypes.data, k[8].ctypes.data, k[9].ctypes.data)
        h = C.c_void_p()
        _check(ctx, load().gpbo_space_create(ctx.handle, C.byref(desc), C.byref(h)))
        self.handle, self.ctx, self.P = h, ctx, P
        self.dim = int(load().gpbo_space_dim(h))

    def encode(self, raw):
        """H0 on the host: raw (n x P) float64 -> encoded (n x d) float32."""
        raw = np.atleast_2d(np.asarray(raw, np.float64))
        out = np.zeros((raw.shape[0], self.dim), np.float32)
        for i in range(raw.shape[0]):
            r = np.ascontiguousarray(raw[i])
            _check(self.ctx, load().gpbo_space_encode(self.handle, r.ctypes.data,
                                                      out[i:].ctypes.data))
        return out

    def sample(self, seed, search, iteration, first, count):
        """H5 on the device: encoded candidates first..first+count-1 (host numpy)."""
        out = np.zeros((count, self.dim), np.float32)
        _check(self.ctx, load().gpbo_space_sample(self.ctx.handle, self.handle, seed, search,
                                                  iteration, first, count, HOST,
                                                  out.ctypes.data))
        return out

    def __del__(self):
        try:
            if self.handle:
                load().gpbo_space_free(self.handle)
                self.handle = None
        except Exception:
            pass


def suggest(ctx, model, spaces, M, seed, iteration, dedup=True):
    """bo_suggest_batch -> (idx int64[S], x_raw list of float64[P_s], ei float32[S])."""
    S = model.S
    arr = (C.c_void_p * S)(*[sp.handle.value for sp in spaces])
    Ma = np.ascontiguousarray(M, dtype=np.int64)
    idx = np.zeros(S, np.int64)
    ei = np.zeros(S, np.float32)
    xr = np.zeros(sum(sp.P for sp in spaces))
    _check(ctx, load().bo_suggest_batch(ctx.handle, model.handle, arr, Ma.ctypes.data, seed,
                                        iteration, int(bool(dedup)), idx.ctypes.data,
                                        xr.ctypes.data, ei.ctypes.data))
    out, o = [], 0
    for sp in spaces:
        out.append(xr[o:o + sp.P])
        o += sp.P
    return idx, out, ei


def version():
    return load().gpbo_version().decode()
