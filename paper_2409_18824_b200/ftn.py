"""Thin ctypes binding of libftn (include/ftn.h): argument marshalling only.

Every computation runs in the CUDA kernels of libftn.so; there is no CPU or
PyTorch fallback.  Importing this module without the built library raises.

Array convention: a Fortran array ``T x(lb1:ub1, ..., lbr:ubr)``
is an ``FArray`` = a CUDA torch tensor of Fortran shape ``(n1, ..., nr)`` whose
strides are the Fortran (column-major) strides, plus its lower bounds.  Sections
are built by ``ftn_desc_section`` (no copy), so negative steps work too.
"""
from __future__ import annotations

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# FTN_LIBFTN: load another build of the library (A/B timing of tuning variants, tools/variants.py)
LIB_PATH = os.environ.get("FTN_LIBFTN") or os.path.join(_HERE, "libftn.so")

I32, I64, F32, F64 = 1, 2, 3, 4
ADD, SUB, MUL, DIV, MULADD = 1, 2, 3, 4, 5
CONTRACT = 1
GEN_U01, GEN_U11, GEN_INT8, GEN_LINEAR, GEN_MOD1024, GEN_RAW = 1, 2, 3, 4, 5, 6
JACOBI_C2 = 0.25
JACOBI_C3 = 1.0 / 6.0  # fl(1/6), R#23

_T2TYPE = {torch.int32: I32, torch.int64: I64, torch.float32: F32, torch.float64: F64}
_TYPE2T = {v: k for k, v in _T2TYPE.items()}
STATUS = ["FTN_OK", "FTN_ERR_NULL", "FTN_ERR_RANK", "FTN_ERR_TYPE", "FTN_ERR_SHAPE", "FTN_ERR_BOUNDS",
          "FTN_ERR_DIM", "FTN_ERR_ALIGN", "FTN_ERR_UNSUPPORTED", "FTN_ERR_WORKSPACE", "FTN_ERR_DEVICE",
          "FTN_ERR_CUDA", "FTN_ERR_NCCL"]


class Dim(ctypes.Structure):
    _fields_ = [("lower_bound", ctypes.c_int64), ("extent", ctypes.c_int64), ("sm", ctypes.c_int64)]


class Desc(ctypes.Structure):
    _fields_ = [("base_addr", ctypes.c_void_p), ("elem_len", ctypes.c_int64), ("rank", ctypes.c_int32),
                ("type", ctypes.c_int32), ("dim", Dim * 3)]


class FtnError(RuntimeError):
    def __init__(self, status: int, call: str, detail: str):
        name = STATUS[status] if 0 <= status < len(STATUS) else str(status)
        super().__init__(f"{call} -> {name}: {detail}")
        self.status = status
        self.name = name


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libftn.so not built at {LIB_PATH}: run `python -m paper_2409_18824_b200.build` "
                          "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    P = ctypes.POINTER(Desc)
    vp, st = ctypes.c_void_p, ctypes.c_int
    i64p = ctypes.POINTER(ctypes.c_int64)
    szp = ctypes.POINTER(ctypes.c_size_t)
    sigs = {
        "ftn_desc_contiguous": [P, vp, ctypes.c_int32, ctypes.c_int32, i64p, i64p],
        "ftn_desc_section": [P, P, i64p, i64p, i64p],
        "ftn_lbound": [P, ctypes.c_int32, i64p],
        "ftn_ubound": [P, ctypes.c_int32, i64p],
        "ftn_size": [P, ctypes.c_int32, i64p],
        "ftn_shape": [P, i64p],
        "ftn_assign": [P, P, vp],
        "ftn_fill": [P, vp, vp],
        "ftn_elemental": [ctypes.c_int32, P, P, P, P, ctypes.c_uint32, vp],
        "ftn_reduce_workspace_size": [P, szp],
        "ftn_sum": [P, vp, vp, ctypes.c_size_t, vp],
        "ftn_maxval": [P, vp, vp, ctypes.c_size_t, vp],
        "ftn_minval": [P, vp, vp, ctypes.c_size_t, vp],
        "ftn_dot_product": [P, P, vp, vp, ctypes.c_size_t, vp],
        "ftn_product": [P, vp, vp, ctypes.c_size_t, vp],
        "ftn_maxval_absdiff": [P, P, vp, vp, ctypes.c_size_t, vp],
        "ftn_jacobi_solve": [P, P, ctypes.c_int64, ctypes.c_int64, ctypes.c_double, ctypes.c_double, vp,
                             ctypes.c_size_t, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_double),
                             ctypes.POINTER(ctypes.c_int32), vp],
        "ftn_sum_dim": [P, ctypes.c_int32, P, vp],
        "ftn_product_dim": [P, ctypes.c_int32, P, vp],
        "ftn_maxval_dim": [P, ctypes.c_int32, P, vp],
        "ftn_minval_dim": [P, ctypes.c_int32, P, vp],
        "ftn_transpose": [P, P, vp],
        "ftn_matmul_workspace_size": [P, P, P, szp],
        "ftn_matmul": [P, P, P, vp, ctypes.c_size_t, vp],
        "ftn_matmul_ex_workspace_size": [P, P, P, ctypes.c_uint32, szp],
        "ftn_matmul_ex": [P, P, P, ctypes.c_uint32, vp, ctypes.c_size_t, vp],
        "ftn_jacobi": [P, P, ctypes.c_int64, ctypes.c_double, ctypes.POINTER(ctypes.c_int32), vp],
        "ftn_jacobi_workspace_size": [P, P, ctypes.c_int64, szp],
        "ftn_jacobi_ws": [P, P, ctypes.c_int64, ctypes.c_double, vp, ctypes.c_size_t, ctypes.POINTER(ctypes.c_int32),
                          vp],
        "ftn_jacobi_solve_workspace_size": [P, P, ctypes.c_int64, ctypes.c_int64, szp],
        "ftn_jacobi_solve_dist": [vp, P, P, ctypes.c_int32, ctypes.c_int64, ctypes.c_int64, ctypes.c_double,
                                  ctypes.c_double, vp, ctypes.c_size_t, ctypes.POINTER(ctypes.c_int64),
                                  ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int32), vp],
        "ftn_comm_unique_id": [ctypes.POINTER(ctypes.c_uint8)],
        "ftn_comm_init": [ctypes.POINTER(vp), ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(ctypes.c_uint8),
                          ctypes.c_int32],
        "ftn_comm_destroy": [vp],
        "ftn_comm_set_overlap": [vp, ctypes.c_int32],
        "ftn_comm_set_sm_reserve": [vp, ctypes.c_int32],
        "ftn_comm_init_virtual": [ctypes.POINTER(vp), ctypes.c_int32, ctypes.POINTER(ctypes.c_int32)],
        "ftn_sum_global": [vp, P, vp, vp, ctypes.c_size_t, vp],
        "ftn_maxval_global": [vp, P, vp, vp, ctypes.c_size_t, vp],
        "ftn_minval_global": [vp, P, vp, vp, ctypes.c_size_t, vp],
        "ftn_dot_product_global": [vp, P, P, vp, vp, ctypes.c_size_t, vp],
        "ftn_jacobi_dist": [vp, P, P, ctypes.c_int64, ctypes.c_double, ctypes.c_int32, ctypes.POINTER(ctypes.c_int32),
                            vp],
        "ftn_jacobi_slab": [P, P, ctypes.c_int32, ctypes.c_double, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, vp],
        "ftn_matmul_colsharded": [vp, P, P, P, vp, ctypes.c_size_t, vp],
        "ftn_bcast": [vp, P, ctypes.c_int32, vp],
        "ftn_gen_fill": [P, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int32, vp],
        "ftn_gen_fill_at": [P, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int32, ctypes.c_uint64, vp],
        "ftn_jacobi_set_fusion": [ctypes.c_int32],
        "ftn_jacobi_host": [vp, vp, P, P, ctypes.c_int64, ctypes.c_double, ctypes.POINTER(ctypes.c_int32), vp],
        "ftn_pw_advection": [P, P, P, P, P, P, P, P, P, P, ctypes.c_double, ctypes.c_double, vp],
        "ftn_tra_adv_workspace_size": [P, szp],
        "ftn_tra_adv": [P, P, P, P, P, P, P, P, P, P, P, P, ctypes.c_int64, vp, ctypes.c_size_t, vp],
    }
    for name, args in sigs.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = st
    L.ftn_jacobi_get_fusion.restype = ctypes.c_int32
    L.ftn_jacobi_get_fusion.argtypes = []
    L.ftn_jacobi_fusion_for.restype = ctypes.c_int32
    L.ftn_jacobi_fusion_for.argtypes = [P]
    L.ftn_jacobi_plan.restype = ctypes.c_int64
    L.ftn_jacobi_plan.argtypes = [ctypes.c_int64, ctypes.c_int32, ctypes.POINTER(ctypes.c_int32), ctypes.c_int64]
    L.ftn_launch_count.restype = ctypes.c_uint64
    L.ftn_launch_count.argtypes = []
    L.ftn_status_string.restype = ctypes.c_char_p
    L.ftn_status_string.argtypes = [ctypes.c_int]
    L.ftn_last_error.restype = ctypes.c_char_p
    L.ftn_last_error.argtypes = []
    return L


lib = _load()


def _call(name: str, *args):
    rc = getattr(lib, name)(*args)
    if rc != 0:
        raise FtnError(rc, name, lib.ftn_last_error().decode())


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


class FArray:
    """A Fortran array (or section) living in a CUDA tensor."""

    def __init__(self, tensor: torch.Tensor, lbounds=None, desc: Desc | None = None):
        self.tensor = tensor  # keeps the storage alive
        if desc is not None:
            self.desc = desc
            return
        if tensor.dtype not in _T2TYPE:
            raise TypeError(f"unsupported dtype {tensor.dtype}")
        r = tensor.dim()
        if r > 3:
            raise ValueError("rank > 3")
        lb = list(lbounds) if lbounds is not None else [1] * r
        d = Desc()
        d.base_addr = tensor.data_ptr()
        d.elem_len = tensor.element_size()
        d.rank = r
        d.type = _T2TYPE[tensor.dtype]
        for k in range(r):
            d.dim[k].lower_bound = lb[k]
            d.dim[k].extent = tensor.shape[k]
            d.dim[k].sm = tensor.stride(k) * tensor.element_size()
        self.desc = d

    # -- construction -------------------------------------------------------------------------
    @staticmethod
    def empty(shape, dtype=torch.float64, lbounds=None, device="cuda") -> "FArray":
        """A contiguous Fortran array of the given Fortran shape (column-major)."""
        shape = tuple(int(s) for s in shape)
        t = torch.empty(shape[::-1], dtype=dtype, device=device).permute(*range(len(shape) - 1, -1, -1))
        return FArray(t, lbounds)

    @staticmethod
    def from_numpy(a, lbounds=None, device="cuda") -> "FArray":
        """Copy a numpy array (any order) into a new contiguous Fortran array."""
        import numpy as np
        fa = FArray.empty(a.shape, dtype=torch.from_numpy(np.zeros(0, dtype=a.dtype)).dtype, lbounds=lbounds,
                          device=device)
        fa.tensor.copy_(torch.from_numpy(np.ascontiguousarray(a)))
        return fa

    @staticmethod
    def scalar(value, dtype=torch.float64, device="cuda") -> "FArray":
        return FArray(torch.tensor(value, dtype=dtype, device=device))

    # -- inquiry ------------------------------------------------------------------------------
    @property
    def rank(self) -> int:
        return self.desc.rank

    @property
    def shape(self):
        return tuple(self.desc.dim[k].extent for k in range(self.rank))

    @property
    def lbounds(self):
        return [self.desc.dim[k].lower_bound for k in range(self.rank)]

    @property
    def strides(self):
        return tuple(self.desc.dim[k].sm for k in range(self.rank))

    @property
    def dtype(self):
        return _TYPE2T[self.desc.type]

    def size(self, dim: int = 0) -> int:
        out = ctypes.c_int64()
        _call("ftn_size", ctypes.byref(self.desc), dim, ctypes.byref(out))
        return out.value

    def lbound(self, dim: int) -> int:
        out = ctypes.c_int64()
        _call("ftn_lbound", ctypes.byref(self.desc), dim, ctypes.byref(out))
        return out.value

    def ubound(self, dim: int) -> int:
        out = ctypes.c_int64()
        _call("ftn_ubound", ctypes.byref(self.desc), dim, ctypes.byref(out))
        return out.value

    def ref(self):
        return ctypes.byref(self.desc)

    def section(self, *triplets) -> "FArray":
        """x(lo:hi:step, ...) with Fortran subscripts; a bare int k means k:k."""
        r = self.rank
        tr = [(t, t, 1) if isinstance(t, int) else (t[0], t[1], t[2] if len(t) > 2 else 1) for t in triplets]
        lo = (ctypes.c_int64 * r)(*[t[0] for t in tr])
        hi = (ctypes.c_int64 * r)(*[t[1] for t in tr])
        st = (ctypes.c_int64 * r)(*[t[2] for t in tr])
        out = Desc()
        _call("ftn_desc_section", ctypes.byref(out), self.ref(), lo, hi, st)
        return FArray(self.tensor, desc=out)

    def whole(self, lbounds=None) -> "FArray":
        """The same memory re-declared with other lower bounds."""
        d = Desc.from_buffer_copy(self.desc)
        for k, lb in enumerate(lbounds or [1] * self.rank):
            d.dim[k].lower_bound = lb
        return FArray(self.tensor, desc=d)

    def view_tensor(self) -> torch.Tensor:
        """A torch view of exactly the described elements (positive strides only)."""
        st = self.tensor.untyped_storage()
        el = self.desc.elem_len
        base = self.tensor.data_ptr() - self.tensor.storage_offset() * el
        off = (self.desc.base_addr or 0) - base
        if self.size() == 0:
            return torch.empty(self.shape, dtype=self.dtype, device=self.tensor.device)
        if off % el or any(s < 0 or s % el for s in self.strides):
            raise ValueError("view_tensor needs positive element-aligned strides")
        t = torch.empty(0, dtype=self.dtype, device=self.tensor.device)
        t.set_(st, off // el, self.shape, tuple(s // el for s in self.strides))
        return t

    def to_numpy(self):
        """Copy the described elements to a host numpy array (Fortran order)."""
        import numpy as np
        if all(s > 0 for s in self.strides):
            return np.asfortranarray(self.view_tensor().cpu().numpy())
        packed = FArray.empty(self.shape, dtype=self.dtype, device=self.tensor.device)
        assign(packed, self)
        return np.asfortranarray(packed.tensor.cpu().numpy())


# ------------------------------------------------------------------------------ workspaces
_ws: dict = {}


def workspace(nbytes: int, device=None, slot: str = "main", stream=None) -> torch.Tensor:
    """Cached device workspace, one per (device, slot, stream): calls on different streams never
    share one, and a buffer is allocated with its stream current so that the caching allocator
    reuses it only in that stream's order after it is replaced."""
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    st = stream if stream is not None else torch.cuda.current_stream(dev)
    key = (dev, slot, st.cuda_stream)
    buf = _ws.get(key)
    if buf is None or buf.numel() < nbytes:
        with torch.cuda.stream(st):
            buf = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=dev)
        _ws[key] = buf
    return buf


def _as_operand(x, like: FArray, stream=None):
    """A Python scalar becomes a rank-0 device operand whose host-to-device copy and lifetime
    are ordered on the stream the kernel runs on (the caching allocator then reuses its block
    only after that stream's later work), not on whatever stream is current."""
    if isinstance(x, FArray):
        return x
    st = stream if stream is not None else torch.cuda.current_stream(like.tensor.device)
    with torch.cuda.stream(st):
        return FArray.scalar(x, dtype=like.dtype, device=like.tensor.device)


# ------------------------------------------------------------------------------ a3
def assign(dst: FArray, src, stream=None):
    """dst = src (src an FArray or a Python scalar)."""
    if not isinstance(src, FArray):
        return fill(dst, src, stream)
    _call("ftn_assign", dst.ref(), src.ref(), _stream(stream))


def fill(dst: FArray, value, stream=None):
    buf = torch.tensor([value], dtype=dst.dtype)
    _call("ftn_fill", dst.ref(), ctypes.c_void_p(buf.data_ptr()), _stream(stream))


def elemental(op: int, dst: FArray, a, b, c=None, contract: bool = False, stream=None):
    """dst = a op b, or dst = a*b + c for op == MULADD (scalars allowed as operands)."""
    a, b = _as_operand(a, dst, stream), _as_operand(b, dst, stream)
    c = _as_operand(c, dst, stream) if c is not None else a
    _call("ftn_elemental", op, dst.ref(), a.ref(), b.ref(), c.ref(), CONTRACT if contract else 0, _stream(stream))


def muladd(dst: FArray, b, c, d, contract: bool = False, stream=None):
    elemental(MULADD, dst, b, c, d, contract, stream)


# ------------------------------------------------------------------------------ a4
def reduce_workspace_size(x: FArray) -> int:
    n = ctypes.c_size_t()
    _call("ftn_reduce_workspace_size", x.ref(), ctypes.byref(n))
    return n.value


def _reduce(name, x: FArray, out=None, stream=None):
    res = out if out is not None else torch.empty((), dtype=x.dtype, device=x.tensor.device)
    ws = workspace(reduce_workspace_size(x), x.tensor.device, "reduce", stream)
    _call(name, x.ref(), ctypes.c_void_p(res.data_ptr()), ctypes.c_void_p(ws.data_ptr()), ws.numel(),
          _stream(stream))
    return res


def sum(x: FArray, out=None, stream=None) -> torch.Tensor:  # noqa: A001 (Fortran name)
    return _reduce("ftn_sum", x, out, stream)


def maxval(x: FArray, out=None, stream=None) -> torch.Tensor:
    return _reduce("ftn_maxval", x, out, stream)


def minval(x: FArray, out=None, stream=None) -> torch.Tensor:
    return _reduce("ftn_minval", x, out, stream)


def product(x: FArray, out=None, stream=None) -> torch.Tensor:
    return _reduce("ftn_product", x, out, stream)


def _reduce_dim(name, x: FArray, dim: int, out: FArray | None = None, stream=None) -> FArray:
    if out is None:
        shape = tuple(e for d, e in enumerate(x.shape) if d != dim - 1)
        out = FArray.empty(shape, dtype=x.dtype, device=x.tensor.device) if shape else \
            FArray(torch.empty((), dtype=x.dtype, device=x.tensor.device))
    _call(name, x.ref(), dim, out.ref(), _stream(stream))
    return out


def sum_dim(x: FArray, dim: int, out=None, stream=None) -> FArray:
    """SUM(x, DIM=dim): sequential fold along dim (R#24)."""
    return _reduce_dim("ftn_sum_dim", x, dim, out, stream)


def product_dim(x: FArray, dim: int, out=None, stream=None) -> FArray:
    return _reduce_dim("ftn_product_dim", x, dim, out, stream)


def maxval_dim(x: FArray, dim: int, out=None, stream=None) -> FArray:
    return _reduce_dim("ftn_maxval_dim", x, dim, out, stream)


def minval_dim(x: FArray, dim: int, out=None, stream=None) -> FArray:
    return _reduce_dim("ftn_minval_dim", x, dim, out, stream)


def dot_product(x: FArray, y: FArray, out=None, stream=None) -> torch.Tensor:
    res = out if out is not None else torch.empty((), dtype=x.dtype, device=x.tensor.device)
    ws = workspace(reduce_workspace_size(x), x.tensor.device, "reduce", stream)
    _call("ftn_dot_product", x.ref(), y.ref(), ctypes.c_void_p(res.data_ptr()), ctypes.c_void_p(ws.data_ptr()),
          ws.numel(), _stream(stream))
    return res


# ------------------------------------------------------------------------------ a5, a6, a7
def transpose(dst: FArray, src: FArray, stream=None):
    _call("ftn_transpose", dst.ref(), src.ref(), _stream(stream))


def matmul_workspace_size(c: FArray, a: FArray, b: FArray) -> int:
    n = ctypes.c_size_t()
    _call("ftn_matmul_workspace_size", c.ref(), a.ref(), b.ref(), ctypes.byref(n))
    return n.value


def matmul(c: FArray, a: FArray, b: FArray, transpose_a: bool = False, transpose_b: bool = False, stream=None,
           force_dmma: bool = False):
    """c = MATMUL(a, b); with transpose_a / transpose_b: MATMUL(TRANSPOSE(a), ...) without a copy.
    Rank-1 operands give the matrix-vector / vector-matrix forms.  Small rank-2 products run the
    sequential-fold kernel unless force_dmma (FTN_MATMUL_FORCE_DMMA) asks for the DMMA path."""
    flags = (1 if transpose_a else 0) | (2 if transpose_b else 0) | (4 if force_dmma else 0)
    if flags:
        n = ctypes.c_size_t()
        _call("ftn_matmul_ex_workspace_size", c.ref(), a.ref(), b.ref(), flags, ctypes.byref(n))
        ws = workspace(n.value, c.tensor.device, "matmul", stream)
        _call("ftn_matmul_ex", c.ref(), a.ref(), b.ref(), flags, ctypes.c_void_p(ws.data_ptr()), ws.numel(),
              _stream(stream))
        return
    ws = workspace(matmul_workspace_size(c, a, b), c.tensor.device, "matmul", stream)
    _call("ftn_matmul", c.ref(), a.ref(), b.ref(), ctypes.c_void_p(ws.data_ptr()), ws.numel(), _stream(stream))


def jacobi(u: FArray, unew: FArray, sweeps: int, coeff: float | None = None, stream=None) -> bool:
    """Run `sweeps` Jacobi sweeps; returns True when the result is in unew."""
    if coeff is None:
        coeff = JACOBI_C2 if u.rank == 2 else JACOBI_C3
    r = ctypes.c_int32()
    n = ctypes.c_size_t()
    _call("ftn_jacobi_workspace_size", u.ref(), unew.ref(), sweeps, ctypes.byref(n))
    if n.value:   # arrays the TMA kernels cannot address: padded copies in a caller workspace
        ws = workspace(n.value, u.tensor.device, "jacobi", stream)
        _call("ftn_jacobi_ws", u.ref(), unew.ref(), sweeps, coeff, ctypes.c_void_p(ws.data_ptr()), ws.numel(),
              ctypes.byref(r), _stream(stream))
    else:
        _call("ftn_jacobi", u.ref(), unew.ref(), sweeps, coeff, ctypes.byref(r), _stream(stream))
    return bool(r.value)


def jacobi_host(host_u: torch.Tensor, host_result: torch.Tensor, u: FArray, unew: FArray, sweeps: int,
                coeff: float | None = None, stream=None) -> bool:
    """ftn_jacobi_host: host_u -> u, u -> unew, `sweeps` sweeps, result -> host_result, on `stream`.
    host_u / host_result: CPU float64 tensors in Fortran (column-major) layout of u's shape."""
    if coeff is None:
        coeff = JACOBI_C2 if u.rank == 2 else JACOBI_C3
    for h in (host_u, host_result):
        col_major = h.permute(*range(h.dim() - 1, -1, -1)).is_contiguous()
        if h.device.type != "cpu" or h.dtype != torch.float64 or tuple(h.shape) != tuple(u.shape) or not col_major:
            raise ValueError("jacobi_host: host buffers must be CPU float64 column-major tensors of u's shape")
    r = ctypes.c_int32()
    _call("ftn_jacobi_host", ctypes.c_void_p(host_u.data_ptr()), ctypes.c_void_p(host_result.data_ptr()), u.ref(),
          unew.ref(), sweeps, coeff, ctypes.byref(r), _stream(stream))
    return bool(r.value)


def pw_advection(su: FArray, sv: FArray, sw: FArray, u: FArray, v: FArray, w: FArray, tzc1: FArray, tzc2: FArray,
                 tzd1: FArray, tzd2: FArray, tcx: float, tcy: float, stream=None) -> None:
    """pw-advection (R#26): su, sv, sw at the interior points."""
    _call("ftn_pw_advection", su.ref(), sv.ref(), sw.ref(), u.ref(), v.ref(), w.ref(), tzc1.ref(), tzc2.ref(),
          tzd1.ref(), tzd2.ref(), tcx, tcy, _stream(stream))


def tra_adv(md: FArray, tsn: FArray, pun: FArray, pvn: FArray, pwn: FArray, umask: FArray, vmask: FArray,
            tmask: FArray, ztfreez: FArray, rnfmsk: FArray, upsmsk: FArray, rnfmsk_z: FArray, iters: int,
            stream=None) -> None:
    """tra-adv (R#28): `iters` iterations of the NEMO tracer-advection nests,
    md updated in place (fields (ji, jj, jk); ztfreez, rnfmsk, upsmsk (ji, jj); rnfmsk_z (jk))."""
    n = ctypes.c_size_t()
    _call("ftn_tra_adv_workspace_size", md.ref(), ctypes.byref(n))
    ws = workspace(n.value, md.tensor.device, "tra_adv", stream)
    _call("ftn_tra_adv", md.ref(), tsn.ref(), pun.ref(), pvn.ref(), pwn.ref(), umask.ref(), vmask.ref(), tmask.ref(),
          ztfreez.ref(), rnfmsk.ref(), upsmsk.ref(), rnfmsk_z.ref(), iters, ctypes.c_void_p(ws.data_ptr()), ws.numel(),
          _stream(stream))


def jacobi_set_fusion(sweeps_per_launch: int):
    """Temporal-blocking factor of the Jacobi kernels (1..12, 0 = the size-dependent default; 3-D uses
    min(T, 2)); results are identical."""
    _call("ftn_jacobi_set_fusion", sweeps_per_launch)


def maxval_absdiff(x: FArray, y: FArray, out=None, stream=None) -> torch.Tensor:
    """MAXVAL(ABS(x - y)) without forming x - y."""
    res = out if out is not None else torch.empty((), dtype=x.dtype, device=x.tensor.device)
    ws = workspace(reduce_workspace_size(x), x.tensor.device, "reduce", stream)
    _call("ftn_maxval_absdiff", x.ref(), y.ref(), ctypes.c_void_p(res.data_ptr()), ctypes.c_void_p(ws.data_ptr()),
          ws.numel(), _stream(stream))
    return res


def jacobi_solve(u: FArray, unew: FArray, max_sweeps: int, check_every: int, tol: float, coeff=None,
                 stream=None) -> tuple[int, float, bool]:
    """Jacobi to convergence (R#25): (sweeps done, last residual, result in unew)."""
    if coeff is None:
        coeff = JACOBI_C2 if u.rank == 2 else JACOBI_C3
    n = ctypes.c_size_t()
    _call("ftn_jacobi_solve_workspace_size", u.ref(), unew.ref(), max_sweeps, check_every, ctypes.byref(n))
    ws = workspace(n.value, u.tensor.device, "solve", stream)
    done, res, new = ctypes.c_int64(), ctypes.c_double(), ctypes.c_int32()
    _call("ftn_jacobi_solve", u.ref(), unew.ref(), max_sweeps, check_every, tol, coeff,
          ctypes.c_void_p(ws.data_ptr()), ws.numel(), ctypes.byref(done), ctypes.byref(res), ctypes.byref(new),
          _stream(stream))
    return done.value, res.value, bool(new.value)


def jacobi_slab(src: FArray, dst: FArray, sweeps: int, halo: int, first: bool, last: bool, coeff=None,
                stream=None):
    """One communication-free local step of the distributed Jacobi (see include/ftn.h)."""
    if coeff is None:
        coeff = JACOBI_C2 if src.rank == 2 else JACOBI_C3
    _call("ftn_jacobi_slab", src.ref(), dst.ref(), sweeps, coeff, halo, int(first), int(last), _stream(stream))


def jacobi_fusion(u: "FArray | None" = None) -> int:
    """The process-wide fusion factor T, or (with u) the sweeps per launch ftn_jacobi uses for u."""
    return int(lib.ftn_jacobi_get_fusion() if u is None else lib.ftn_jacobi_fusion_for(u.ref()))


def jacobi_plan(sweeps: int, T: int | None = None) -> list[int]:
    """Sweeps per launch that ftn_jacobi uses for a rank-2 TMA-able array (ftn_jacobi_plan)."""
    T = jacobi_fusion() if T is None else T
    n = lib.ftn_jacobi_plan(sweeps, T, None, 0)
    buf = (ctypes.c_int32 * max(n, 1))()
    lib.ftn_jacobi_plan(sweeps, T, buf, n)
    return list(buf[:n])


def gen_fill(dst: FArray, seed: int, array_id: int, mode: int, stream=None, t0: int = 0):
    """Seeded synthetic values; t0: index of dst's first element in the sequence."""
    _call("ftn_gen_fill_at", dst.ref(), seed & 0xFFFFFFFFFFFFFFFF, array_id, mode, t0, _stream(stream))


def launch_count() -> int:
    return int(lib.ftn_launch_count())


# ------------------------------------------------------------------------------ a8
class Comm:
    """A communicator for one rank: NCCL (bootstrapped through torch.distributed), or one of
    the virtual ranks of this process (Comm.virtual; each rank driven by its own thread)."""

    def __init__(self, nranks: int, rank: int, uid: bytes | None, device: int, handle=None):
        self.nranks, self.rank, self.device = nranks, rank, device
        if handle is not None:
            self.handle = handle
            return
        buf = (ctypes.c_uint8 * 128).from_buffer_copy(uid)
        self.handle = ctypes.c_void_p()
        _call("ftn_comm_init", ctypes.byref(self.handle), nranks, rank, buf, device)

    @staticmethod
    def virtual(nranks: int, devices=None) -> list["Comm"]:
        """nranks virtual ranks in this process (ftn_comm_init_virtual), all on the current
        device unless `devices` lists one device per rank."""
        if devices is None:
            devices = [torch.cuda.current_device()] * nranks
        arr = (ctypes.c_void_p * nranks)()
        devs = (ctypes.c_int32 * nranks)(*devices)
        _call("ftn_comm_init_virtual", arr, nranks, devs)
        return [Comm(nranks, r, None, devices[r], handle=ctypes.c_void_p(arr[r])) for r in range(nranks)]

    @staticmethod
    def unique_id() -> bytes:
        buf = (ctypes.c_uint8 * 128)()
        _call("ftn_comm_unique_id", buf)
        return bytes(buf)

    @staticmethod
    def from_torch_distributed(device: int) -> "Comm":
        import torch.distributed as dist
        rank, n = dist.get_rank(), dist.get_world_size()
        obj = [Comm.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return Comm(n, rank, obj[0], device)

    def destroy(self):
        if self.handle:
            _call("ftn_comm_destroy", self.handle)
            self.handle = ctypes.c_void_p()

    def set_overlap(self, mode: int):
        """Halo exchange / interior sweep overlap in jacobi(): 0 off, 1 when nranks > 1, 2 always."""
        _call("ftn_comm_set_overlap", self.handle, mode)

    def set_sm_reserve(self, sms: int):
        """SMs the side-stream interior sweeps leave free for the exchange kernels."""
        _call("ftn_comm_set_sm_reserve", self.handle, sms)

    def _ws(self, x: FArray, stream=None) -> torch.Tensor:
        return workspace(reduce_workspace_size(x) + 8 * (self.nranks + 1) + 64, x.tensor.device, "global", stream)

    def _global(self, name, x: FArray, out=None, stream=None):
        res = out if out is not None else torch.empty((), dtype=x.dtype, device=x.tensor.device)
        ws = self._ws(x, stream)
        _call(name, self.handle, x.ref(), ctypes.c_void_p(res.data_ptr()), ctypes.c_void_p(ws.data_ptr()),
              ws.numel(), _stream(stream))
        return res

    def sum(self, x, out=None, stream=None):
        return self._global("ftn_sum_global", x, out, stream)

    def maxval(self, x, out=None, stream=None):
        return self._global("ftn_maxval_global", x, out, stream)

    def minval(self, x, out=None, stream=None):
        return self._global("ftn_minval_global", x, out, stream)

    def dot_product(self, x, y, out=None, stream=None):
        res = out if out is not None else torch.empty((), dtype=x.dtype, device=x.tensor.device)
        ws = self._ws(x, stream)
        _call("ftn_dot_product_global", self.handle, x.ref(), y.ref(), ctypes.c_void_p(res.data_ptr()),
              ctypes.c_void_p(ws.data_ptr()), ws.numel(), _stream(stream))
        return res

    def jacobi(self, u: FArray, unew: FArray, sweeps: int, coeff=None, halo: int = 1, stream=None) -> bool:
        """Distributed sweeps of this rank's slab (halo planes per side)."""
        if coeff is None:
            coeff = JACOBI_C2 if u.rank == 2 else JACOBI_C3
        r = ctypes.c_int32()
        _call("ftn_jacobi_dist", self.handle, u.ref(), unew.ref(), sweeps, coeff, halo, ctypes.byref(r),
              _stream(stream))
        return bool(r.value)

    def jacobi_solve(self, u: FArray, unew: FArray, max_sweeps: int, check_every: int, tol: float, coeff=None,
                     halo: int = 1, stream=None) -> tuple[int, float, bool]:
        """Distributed Jacobi to convergence (ftn_jacobi_solve_dist): (sweeps done, global residual,
        result in unew), identical on every rank."""
        if coeff is None:
            coeff = JACOBI_C2 if u.rank == 2 else JACOBI_C3
        ws = workspace(8 * (self.nranks + 2) + reduce_workspace_size(u), u.tensor.device, "solve_dist", stream)
        done, res, new = ctypes.c_int64(), ctypes.c_double(), ctypes.c_int32()
        _call("ftn_jacobi_solve_dist", self.handle, u.ref(), unew.ref(), halo, max_sweeps, check_every, tol, coeff,
              ctypes.c_void_p(ws.data_ptr()), ws.numel(), ctypes.byref(done), ctypes.byref(res), ctypes.byref(new),
              _stream(stream))
        return done.value, res.value, bool(new.value)

    def matmul(self, c_local: FArray, a_full: FArray, b_local: FArray, stream=None):
        ws = workspace(matmul_workspace_size(c_local, a_full, b_local), c_local.tensor.device, "matmul", stream)
        _call("ftn_matmul_colsharded", self.handle, c_local.ref(), a_full.ref(), b_local.ref(),
              ctypes.c_void_p(ws.data_ptr()), ws.numel(), _stream(stream))

    def bcast(self, x: FArray, root: int = 0, stream=None):
        _call("ftn_bcast", self.handle, x.ref(), root, _stream(stream))
