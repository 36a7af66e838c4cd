"""ctypes binding of include/lsba.h (argument marshalling only; every step runs in liblsba.so).

Device buffers are torch CUDA float64 tensors (row-major n_local x s, contiguous); host
buffers are numpy arrays.  Streams: the torch current stream of the tensor's device.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
library_path = os.path.join(_HERE, "liblsba.so")

if not os.path.exists(library_path):
    raise ImportError(f"{library_path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                      "(paper_2208_09899_b200/build.sh). There is no CPU fallback.")
lib = C.CDLL(library_path)

LSBA_OK, LSBA_E_ARG, LSBA_E_CUDA, LSBA_E_NCCL, LSBA_E_OOM, LSBA_E_STATE, LSBA_E_NUMERIC = range(7)
LSBA_IP_CLASSICAL, LSBA_IP_GLOBAL = 0, 1
(LSBA_SKEL_BCGS_PIP, LSBA_SKEL_BMGS_CWY, LSBA_SKEL_BMGS_ICWY, LSBA_SKEL_BMGS, LSBA_SKEL_BCGS_PIO,
 LSBA_SKEL_BCGS_IROLS) = 0, 1, 2, 3, 4, 5
_SKEL = {"pip": 0, "cwy": 1, "icwy": 2, "bmgs": 3, "pio": 4, "irols": 5, 0: 0, 1: 1, 2: 2, 3: 3, 4: 4, 5: 5}
LSBA_CONVERGED, LSBA_MAX_RESTARTS, LSBA_DEAD = 0, 1, 2
KERNEL_IDS = dict(spmm=0, gram=1, gram_finalize=2, small_step=3, project=4, cycle_solve=5,
                  combine=6, residual=7, halo_pack=8, misc=9, step_update=10, ilu_solve=11)
_IP = {"cl": LSBA_IP_CLASSICAL, "gl": LSBA_IP_GLOBAL, 0: 0, 1: 1}


class StepInfo(C.Structure):
    _fields_ = [("k", C.c_int32), ("chol_flag", C.c_int32), ("cond_est", C.c_double),
                ("res_est", C.c_double), ("res_est_fom", C.c_double), ("proj_singular", C.c_int32),
                ("pad_", C.c_int32)]


class SolveInfo(C.Structure):
    _fields_ = [("outcome", C.c_int32), ("cycles", C.c_int32), ("restarts", C.c_int32),
                ("iterations", C.c_int32), ("attempted_steps", C.c_int32),
                ("nan_flags", C.c_int32), ("cond_restarts", C.c_int32), ("happy", C.c_int32),
                ("false_convergences", C.c_int32), ("m_final", C.c_int32),
                ("syncs", C.c_int64), ("matvecs", C.c_int64), ("basis_evals", C.c_int64),
                ("kernel_launches", C.c_int64),
                ("res_est", C.c_double), ("true_relres", C.c_double), ("seconds", C.c_double),
                ("gram_blocks", C.c_int64)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


_vp, _i32, _i64, _d = C.c_void_p, C.c_int32, C.c_int64, C.c_double

# lsba_allocator (include/lsba.h): the caller-owned workspace variant of lsba_create
_ALLOC_FN = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_int32, C.c_void_p, C.c_void_p)
_FREE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p)


class Allocator(C.Structure):
    _fields_ = [("alloc", _ALLOC_FN), ("free", _FREE_FN), ("user", C.c_void_p)]


def torch_allocator():
    """An lsba_allocator backed by PyTorch's caching allocator (torch owns the workspace)."""
    import torch

    def _alloc(nbytes, device, stream, user):
        try:
            return torch.cuda.caching_allocator_alloc(int(nbytes), int(device), int(stream or 0))
        except Exception:           # (OOM -> NULL -> LSBA_E_OOM)
            return None

    def _free(ptr, device, stream, user):
        torch.cuda.caching_allocator_delete(int(ptr))

    a = Allocator(_ALLOC_FN(_alloc), _FREE_FN(_free), None)
    a._keep = (_alloc, _free)      # the Python callables must outlive the context
    return a
_sigs = {
    "lsba_get_unique_id": [_vp],
    "lsba_create": [C.POINTER(_vp), _i64, _i32, _i32, _vp, _vp, _vp, _i64, _i64, _i32, _i32, _vp, _i32, _vp],
    "lsba_destroy": [_vp],
    "lsba_loopback_create": [_i32, C.POINTER(_vp)],
    "lsba_loopback_destroy": [_vp],
    "lsba_create_loopback": [C.POINTER(_vp), _i64, _i32, _i32, _vp, _vp, _vp, _i64, _i64, _i32, _i32, _vp, _i32, _vp],
    "lsba_create_with_allocator": [C.POINTER(_vp), _i64, _i32, _i32, _vp, _vp, _vp, _i64, _i64, _i32, _i32, _vp,
                                   _i32, _vp, _vp],
    "lsba_arnoldi_begin": [_vp, _vp, C.c_int, C.POINTER(_i32)],
    "lsba_block_arnoldi_step": [_vp, C.POINTER(StepInfo)],
    "lsba_copy_hessenberg": [_vp, _vp, _i32],
    "lsba_projected_solve": [_vp, _i32, _vp, _vp],
    "lsba_copy_beta": [_vp, _vp],
    "lsba_copy_basis_block": [_vp, _i32, _vp],
    "lsba_bgmres_solve": [_vp, _vp, _vp, _i32, _d, _i32, C.c_int, C.c_int, _d, C.POINTER(SolveInfo)],
    "lsba_bfom_solve": [_vp, _vp, _vp, _i32, _d, _i32, C.c_int, C.c_int, _d, C.POINTER(SolveInfo)],
    "lsba_solve_host": [_vp, _vp, _vp, _i32, _d, _i32, _i32, C.c_int, _d, C.POINTER(SolveInfo)],
    "lsba_spmm": [_vp, _vp, _vp],
    "lsba_block_inner_product": [_vp, _vp, _i32, _vp, C.c_int, _vp],
    "lsba_set_force_flag": [_vp, _i32],
    "lsba_set_force_singular": [_vp, _i32],
    "lsba_set_basis_block": [_vp, _i32, _vp],
    "lsba_basis_inner_product": [_vp, _i32, _i32, _i32, _i32, _i32, _vp],
    "lsba_set_kernel_variant": [_vp, _i32],
    "lsba_set_skeleton": [_vp, C.c_int],
    "lsba_profile_enable": [_vp, _i32],
    "lsba_profile_read": [_vp, _i32, C.POINTER(_i64), C.POINTER(_d), C.POINTER(_d)],
    "lsba_profile_timeline": [_vp, _vp, _vp, _vp, _i64, C.POINTER(_i64)],
    "lsba_launch_count": [_vp, C.POINTER(_i64)],
    "lsba_workspace_bytes": [_vp, C.POINTER(_i64)],
    "lsba_ghost_plan": [_i64, _i64, _vp, _i64, _vp, _i32, _vp, _vp, C.POINTER(_i64), _vp],
    "lsba_csr_validate": [_i64, _i64, _vp, _vp, C.POINTER(C.c_char_p)],
    "lsba_ilu0_setup": [_vp, _i32],
    "lsba_ilu0_apply": [_vp, _vp, _vp],
    "lsba_copy_ilu0_factors": [_vp, _vp, _i64, _vp],
    "lsba_status_str": [C.c_int],
    "lsba_last_error": [_vp],
}
for _name, _args in _sigs.items():
    _f = getattr(lib, _name)
    _f.argtypes = _args
    _f.restype = C.c_char_p if _name in ("lsba_status_str", "lsba_last_error") else C.c_int


class LsbaError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{lib.lsba_status_str(status).decode()}: {msg}")
        self.status = status


def lsba_status_str(st: int) -> str:
    return lib.lsba_status_str(st).decode()


def lsba_last_error(ctx) -> str:
    return lib.lsba_last_error(ctx).decode()


def _check(st, ctx=None):
    if st != LSBA_OK:
        raise LsbaError(st, lsba_last_error(ctx) if ctx else "")


def _dptr(t, name="buffer"):
    """Device pointer of a contiguous float64 CUDA tensor."""
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA torch tensor")
    if t.dtype != torch.float64 or not t.is_contiguous():
        raise TypeError(f"{name} must be contiguous float64")
    return C.c_void_p(t.data_ptr())


def _hptr(a):
    return a.ctypes.data_as(C.c_void_p)


# ------------------------------------------------------------------ thin wrappers (same names)
def lsba_get_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    _check(lib.lsba_get_unique_id(buf))
    return bytes(buf)


def lsba_loopback_create(nranks):
    """A loopback group (P ranks as host threads on one device; testing only)."""
    g = C.c_void_p()
    _check(lib.lsba_loopback_create(int(nranks), C.byref(g)))
    return g


def lsba_loopback_destroy(group):
    _check(lib.lsba_loopback_destroy(group))


def lsba_create_loopback(n, s, m_max, row_ptr, col_idx, vals, row_begin, row_end, rank, nranks, group,
                         device=0, stream=None):
    return lsba_create(n, s, m_max, row_ptr, col_idx, vals, row_begin, row_end, rank, nranks,
                       device=device, stream=stream, loopback=group)


def lsba_create_with_allocator(n, s, m_max, row_ptr, col_idx, vals, row_begin, row_end, rank, nranks,
                               nccl_id, device, stream, allocator):
    return lsba_create(n, s, m_max, row_ptr, col_idx, vals, row_begin, row_end, rank, nranks, nccl_id,
                       device, stream, allocator=allocator)


def lsba_create(n, s, m_max, row_ptr, col_idx, vals, row_begin=0, row_end=None, rank=0, nranks=1,
                nccl_id=None, device=0, stream=None, loopback=None, allocator=None):
    """row_ptr/col_idx/vals: host numpy (int64 / int32 global cols / float64) for the local rows.
    loopback: a group from lsba_loopback_create (then nccl_id is not used).
    allocator: an Allocator (e.g. torch_allocator()) that owns the workspace."""
    row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int64)
    col_idx = np.ascontiguousarray(col_idx, dtype=np.int32)
    vals = np.ascontiguousarray(vals, dtype=np.float64)
    if row_end is None:
        row_end = n
    ctx = C.c_void_p()
    idbuf = None
    if nccl_id is not None:
        idbuf = (C.c_uint8 * 128).from_buffer_copy(nccl_id)
    if allocator is not None:
        st = lib.lsba_create_with_allocator(C.byref(ctx), int(n), int(s), int(m_max), _hptr(row_ptr), _hptr(col_idx),
                                            _hptr(vals), int(row_begin), int(row_end), int(rank), int(nranks), idbuf,
                                            int(device), C.c_void_p(stream or 0), C.byref(allocator))
    elif loopback is not None:
        st = lib.lsba_create_loopback(C.byref(ctx), int(n), int(s), int(m_max), _hptr(row_ptr), _hptr(col_idx),
                                      _hptr(vals), int(row_begin), int(row_end), int(rank), int(nranks),
                                      loopback, int(device), C.c_void_p(stream or 0))
    else:
        st = lib.lsba_create(C.byref(ctx), int(n), int(s), int(m_max), _hptr(row_ptr), _hptr(col_idx),
                             _hptr(vals), int(row_begin), int(row_end), int(rank), int(nranks), idbuf,
                             int(device), C.c_void_p(stream or 0))
    if st != LSBA_OK:
        msg = lsba_last_error(ctx) if ctx else ""
        if ctx:
            lib.lsba_destroy(ctx)
        raise LsbaError(st, msg)
    return ctx


def lsba_destroy(ctx):
    _check(lib.lsba_destroy(ctx))


def lsba_arnoldi_begin(ctx, B, ip="cl") -> int:
    flag = C.c_int32(0)
    _check(lib.lsba_arnoldi_begin(ctx, _dptr(B, "B"), _IP[ip], C.byref(flag)), ctx)
    return flag.value


def lsba_block_arnoldi_step(ctx) -> StepInfo:
    info = StepInfo()
    _check(lib.lsba_block_arnoldi_step(ctx, C.byref(info)), ctx)
    return info


def lsba_copy_hessenberg(ctx, nrows, ncols):
    H = np.zeros((ncols, nrows))        # column-major (ld = nrows) == C-order transpose
    _check(lib.lsba_copy_hessenberg(ctx, _hptr(H), int(nrows)), ctx)
    return H.T.copy()


def lsba_projected_solve(ctx, k, b, fom=False):
    Xi = np.zeros((k * b, b))
    Z = np.zeros(((k + 1) * b, b))
    _check(lib.lsba_projected_solve(ctx, 1 if fom else 0, _hptr(Xi), _hptr(Z)), ctx)
    return Xi, Z


def lsba_copy_beta(ctx, b):
    out = np.zeros((b, b))
    _check(lib.lsba_copy_beta(ctx, _hptr(out)), ctx)
    return out.T.copy()


def lsba_copy_basis_block(ctx, j, dst):
    _check(lib.lsba_copy_basis_block(ctx, int(j), _dptr(dst, "dst")), ctx)
    return dst


def _solve(fn, ctx, B, X, m, tol, max_restarts, ip, cond_threshold, skel):
    info = SolveInfo()
    _check(fn(ctx, _dptr(B, "B"), _dptr(X, "X"), int(m), float(tol), int(max_restarts),
              _SKEL[skel], _IP[ip], float(cond_threshold), C.byref(info)), ctx)
    return info


def lsba_bgmres_solve(ctx, B, X, m, tol, max_restarts, ip="cl", cond_threshold=float("inf"), skel="pip"):
    return _solve(lib.lsba_bgmres_solve, ctx, B, X, m, tol, max_restarts, ip, cond_threshold, skel)


def lsba_bfom_solve(ctx, B, X, m, tol, max_restarts, ip="cl", cond_threshold=float("inf"), skel="pip"):
    return _solve(lib.lsba_bfom_solve, ctx, B, X, m, tol, max_restarts, ip, cond_threshold, skel)


def lsba_set_skeleton(ctx, skel):
    _check(lib.lsba_set_skeleton(ctx, _SKEL[skel]), ctx)


def lsba_solve_host(ctx, B, X, m, tol, max_restarts, fom=False, ip="cl", cond_threshold=float("inf")):
    """B, X: host numpy float64 C-contiguous (n_local x s); X is X0 on entry, X on exit."""
    assert B.flags.c_contiguous and X.flags.c_contiguous and X.dtype == np.float64 and B.dtype == np.float64
    info = SolveInfo()
    _check(lib.lsba_solve_host(ctx, _hptr(B), _hptr(X), int(m), float(tol), int(max_restarts),
                               1 if fom else 0, _IP[ip], float(cond_threshold), C.byref(info)), ctx)
    return info


def lsba_spmm(ctx, V, W):
    _check(lib.lsba_spmm(ctx, _dptr(V, "V"), _dptr(W, "W")), ctx)
    return W


def lsba_block_inner_product(ctx, V, nblocks, Y, ip="cl", s=None):
    s = s if s is not None else Y.shape[-1]
    E = nblocks * s * s if _IP[ip] == LSBA_IP_CLASSICAL else nblocks
    G = np.zeros(E)
    _check(lib.lsba_block_inner_product(ctx, _dptr(V, "V"), int(nblocks), _dptr(Y, "Y"), _IP[ip], _hptr(G)), ctx)
    return G.reshape(nblocks * s, s) if _IP[ip] == LSBA_IP_CLASSICAL else G


def lsba_ilu0_setup(ctx, enable=True):
    _check(lib.lsba_ilu0_setup(ctx, 1 if enable else 0), ctx)


def lsba_ilu0_apply(ctx, X, Y):
    _check(lib.lsba_ilu0_apply(ctx, _dptr(X, "X"), _dptr(Y, "Y")), ctx)
    return Y


def lsba_copy_ilu0_factors(ctx, nnz):
    """(factor values (nnz,), (levels of L, levels of U)); nnz = 0 fetches the levels only."""
    lu = np.zeros(max(int(nnz), 1))
    lev = np.zeros(2, dtype=np.int32)
    _check(lib.lsba_copy_ilu0_factors(ctx, _hptr(lu) if nnz > 0 else None, int(nnz), _hptr(lev)), ctx)
    return lu[:nnz], (int(lev[0]), int(lev[1]))


def lsba_set_force_flag(ctx, k):
    _check(lib.lsba_set_force_flag(ctx, int(k)), ctx)


def lsba_set_basis_block(ctx, j, src):
    _check(lib.lsba_set_basis_block(ctx, int(j), _dptr(src, "src")), ctx)


def lsba_basis_inner_product(ctx, j0, nblocks, y, y2=0, ip="cl", s=None):
    """<[V_j0 .. V_{j0+nblocks-1}], V_y (, V_y2)> over basis slots by the shipped Gram kernels.
    Classical: (nblocks s) x (s or 2s); global: (nblocks,) or (nblocks, 2)."""
    ipc = _IP[ip]
    if s is None:
        raise ValueError("s is required")
    w = 2 if y2 else 1
    E = nblocks * (1 if ipc == LSBA_IP_GLOBAL else s * s) * w
    G = np.zeros(E)
    _check(lib.lsba_basis_inner_product(ctx, int(j0), int(nblocks), int(y), int(y2), ipc, _hptr(G)), ctx)
    if ipc == LSBA_IP_GLOBAL:
        return G.reshape(nblocks, w) if w == 2 else G
    return G.reshape(nblocks * s, w * s)


def lsba_set_force_singular(ctx, cycle):
    _check(lib.lsba_set_force_singular(ctx, int(cycle)), ctx)


def lsba_set_kernel_variant(ctx, variant):
    _check(lib.lsba_set_kernel_variant(ctx, int(variant)), ctx)


def lsba_profile_enable(ctx, enable=True):
    _check(lib.lsba_profile_enable(ctx, 1 if enable else 0), ctx)


def lsba_profile_read(ctx, kid):
    n, ms, by = C.c_int64(), C.c_double(), C.c_double()
    kid = KERNEL_IDS[kid] if isinstance(kid, str) else kid
    _check(lib.lsba_profile_read(ctx, int(kid), C.byref(n), C.byref(ms), C.byref(by)), ctx)
    return n.value, ms.value, by.value


def lsba_profile_timeline(ctx):
    """[(kernel name, start ms, end ms)] of the recorded launches in issue order."""
    n = C.c_int64()
    _check(lib.lsba_profile_timeline(ctx, None, None, None, 0, C.byref(n)), ctx)
    kids = np.zeros(max(n.value, 1), dtype=np.int32)
    t0 = np.zeros(max(n.value, 1))
    t1 = np.zeros(max(n.value, 1))
    _check(lib.lsba_profile_timeline(ctx, _hptr(kids), _hptr(t0), _hptr(t1), n.value, C.byref(n)), ctx)
    names = {v: k for k, v in KERNEL_IDS.items()}
    return [(names.get(int(k), str(k)), float(a), float(b)) for k, a, b in zip(kids[:n.value], t0, t1)]


def lsba_launch_count(ctx):
    n = C.c_int64()
    _check(lib.lsba_launch_count(ctx, C.byref(n)), ctx)
    return n.value


def lsba_workspace_bytes(ctx):
    n = C.c_int64()
    _check(lib.lsba_workspace_bytes(ctx, C.byref(n)), ctx)
    return n.value


def lsba_ghost_plan(row_begin, row_end, col_idx, part):
    """Host-only ghost plan (no GPU needed).  Returns (col_local, ghost_global, recv_counts)."""
    col_idx = np.ascontiguousarray(col_idx, dtype=np.int32)
    part = np.ascontiguousarray(part, dtype=np.int64)
    nnz = col_idx.size
    col_local = np.zeros(max(nnz, 1), dtype=np.int32)
    ghost = np.zeros(max(nnz, 1), dtype=np.int64)
    recv = np.zeros(part.size - 1, dtype=np.int64)
    ng = C.c_int64()
    st = lib.lsba_ghost_plan(int(row_begin), int(row_end), _hptr(col_idx), nnz, _hptr(part),
                             part.size - 1, _hptr(col_local), _hptr(ghost), C.byref(ng), _hptr(recv))
    _check(st)
    return col_local[:nnz], ghost[: ng.value], recv


def lsba_csr_validate(n_rows, n_cols, row_ptr, col_idx):
    row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int64)
    col_idx = np.ascontiguousarray(col_idx, dtype=np.int32)
    msg = C.c_char_p()
    st = lib.lsba_csr_validate(int(n_rows), int(n_cols), _hptr(row_ptr), _hptr(col_idx), C.byref(msg))
    return st, (msg.value or b"").decode()


# ------------------------------------------------------------------ convenience object
class Context:
    """RAII wrapper: one context (one rank's rows) on one device."""

    def __init__(self, n, s, m_max, row_ptr, col_idx, vals, row_begin=0, row_end=None, rank=0,
                 nranks=1, nccl_id=None, device=None, stream=None, loopback=None, allocator=None):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2208_09899_b200 needs a CUDA device (no CPU fallback)")
        device = torch.cuda.current_device() if device is None else device
        if stream is None:
            stream = torch.cuda.current_stream(device).cuda_stream
        self.n, self.s, self.m_max = n, s, m_max
        self.row_begin = row_begin
        self.row_end = n if row_end is None else row_end
        self.n_local = self.row_end - self.row_begin
        self.device = device
        # allocator="torch": PyTorch's caching allocator owns the workspace (lsba_create_with_allocator)
        self.allocator = torch_allocator() if allocator == "torch" else allocator
        self.ctx = lsba_create(n, s, m_max, row_ptr, col_idx, vals, row_begin, self.row_end, rank,
                               nranks, nccl_id, device, stream, loopback, self.allocator)

    def close(self):
        if getattr(self, "ctx", None):
            lsba_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # pass-throughs
    def begin(self, B, ip="cl"):
        return lsba_arnoldi_begin(self.ctx, B, ip)

    def step(self):
        return lsba_block_arnoldi_step(self.ctx)

    def hessenberg(self, k, b):
        return lsba_copy_hessenberg(self.ctx, (k + 1) * b, k * b)

    def beta(self, b):
        return lsba_copy_beta(self.ctx, b)

    def basis_block(self, j):
        import torch
        out = torch.empty((self.n_local, self.s), dtype=torch.float64, device=f"cuda:{self.device}")
        return lsba_copy_basis_block(self.ctx, j, out)

    def spmm(self, V):
        import torch
        W = torch.empty_like(V)
        return lsba_spmm(self.ctx, V, W)

    def solve(self, B, X, m, tol, max_restarts, ip="cl", mod="gmres", cond_threshold=float("inf"), skel="pip",
              prec=None):
        """prec=None: the plain operator; prec="ilu0": left ILU(0) (factored on first use)."""
        if prec not in (None, "ilu0"):
            raise ValueError(f"unknown preconditioner {prec!r}")
        lsba_ilu0_setup(self.ctx, prec == "ilu0")
        fn = lsba_bgmres_solve if mod == "gmres" else lsba_bfom_solve
        return fn(self.ctx, B, X, m, tol, max_restarts, ip, cond_threshold, skel)

    def ilu0_apply(self, X):
        import torch
        Y = torch.empty_like(X)
        return lsba_ilu0_apply(self.ctx, X, Y)
