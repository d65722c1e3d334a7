"""CPU oracle for the Fortran array statements of arXiv 2409.18824 -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  It shares no code with the
CUDA library (``paper_2409_18824_b200``) and never imports it.

The arithmetic lives in ``ftn_oracle.c`` (plain sequential C, -O2
-ffp-contract=off); this module only marshals numpy arrays into the oracle's own
descriptor struct.  A Fortran array ``T x(lb1:ub1, ..., lbr:ubr)`` is a numpy
array of shape ``(n1, ..., nr)`` whose byte strides are the Fortran strides
(``order='F'`` for a whole array; any view for a section), plus its lbounds.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ftn_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

I32, I64, F32, F64 = 1, 2, 3, 4
ADD, SUB, MUL, DIV, MULADD = 1, 2, 3, 4, 5
SUM, MAX, MIN, PROD = 0, 1, 2, 3
R_CHUNK = 65536  # DESIGN.md section 4.2, step 2

_NP2TYPE = {np.dtype(np.int32): I32, np.dtype(np.int64): I64,
            np.dtype(np.float32): F32, np.dtype(np.float64): F64}


def build(openmp: bool = True, sanitize: bool = False) -> str:
    """Compile liboracle.so with gcc (-O2 -ffp-contract=off; no -ffast-math).  sanitize=True
    builds liboracle_san.so instead: AddressSanitizer + UndefinedBehaviorSanitizer, errors fatal,
    no OpenMP (tests/test_oracle_sanitized.py loads it through FTN_ORACLE_LIB)."""
    out = _LIB if not sanitize else os.path.join(_HERE, "liboracle_san.so")
    cmd = ["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared", "-std=gnu11",
           "-Wall", _SRC, "-o", out + ".tmp", "-lm"]
    if sanitize:
        cmd[1:1] = ["-g", "-fno-omit-frame-pointer", "-fsanitize=address,undefined", "-fno-sanitize-recover=all"]
    elif openmp:
        cmd.insert(1, "-fopenmp")
    subprocess.run(cmd, check=True)
    os.replace(out + ".tmp", out)
    return out


class _Dim(ctypes.Structure):
    _fields_ = [("lb", ctypes.c_int64), ("ext", ctypes.c_int64), ("sm", ctypes.c_int64)]


class _Array(ctypes.Structure):
    _fields_ = [("base", ctypes.c_void_p), ("type", ctypes.c_int32), ("rank", ctypes.c_int32),
                ("dim", _Dim * 3)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        path = os.environ.get("FTN_ORACLE_LIB")   # e.g. the sanitizer build
        if path is None:
            if (not os.path.exists(_LIB)) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
                build()
            path = _LIB
        L = ctypes.CDLL(path)
        P = ctypes.POINTER(_Array)
        i64p = ctypes.POINTER(ctypes.c_int64)
        dp = ctypes.POINTER(ctypes.c_double)
        sig = {
            "orc_section": (ctypes.c_int, [P, i64p, i64p, i64p, P]),
            "orc_triplet_indices": (ctypes.c_int64, [ctypes.c_int64] * 3 + [i64p, ctypes.c_int64]),
            "orc_element_offset": (ctypes.c_int64, [P, i64p]),
            "orc_elemental": (ctypes.c_int, [ctypes.c_int32, P, P, P, P, ctypes.c_int32]),
            "orc_assign": (ctypes.c_int, [P, P]),
            "orc_sum_seq_f64": (ctypes.c_double, [P]),
            "orc_sum_i64": (ctypes.c_int64, [P]),
            "orc_sum_i32": (ctypes.c_int32, [P]),
            "orc_sum_exact_f64": (ctypes.c_double, [P]),
            "orc_sum_abs_f64": (ctypes.c_double, [P]),
            "orc_fsum": (ctypes.c_double, [dp, ctypes.c_int64]),
            "orc_tree_combine": (ctypes.c_double, [dp, ctypes.c_int64, ctypes.c_int32]),
            "orc_orderR_partials": (None, [dp, ctypes.c_int64, ctypes.c_int32, dp]),
            "orc_reduce_orderR_f64": (ctypes.c_double, [P, ctypes.c_int32]),
            "orc_maxval_f64": (ctypes.c_double, [P]),
            "orc_minval_f64": (ctypes.c_double, [P]),
            "orc_maxval_int": (ctypes.c_int64, [P]),
            "orc_minval_int": (ctypes.c_int64, [P]),
            "orc_dot_products_f64": (ctypes.c_int, [P, P, dp]),
            "orc_dot_exact_f64": (ctypes.c_int, [P, P, dp, dp]),
            "orc_transpose": (ctypes.c_int, [P, P]),
            "orc_matmul_f64": (ctypes.c_int, [P, P, P, P]),
            "orc_matmul_element_f64": (ctypes.c_double, [P, P, ctypes.c_int64, ctypes.c_int64, dp]),
            "orc_jacobi_f64": (ctypes.c_int, [P, P, ctypes.c_int64, ctypes.c_double,
                                              ctypes.POINTER(ctypes.c_int32)]),
            "orc_product_seq_f64": (ctypes.c_double, [P]),
            "orc_product_int": (ctypes.c_int64, [P]),
            "orc_reduce_dim": (ctypes.c_int, [P, ctypes.c_int32, ctypes.c_int32, P]),
            "orc_matvec_f64": (ctypes.c_int, [P, P, P, P]),
            "orc_maxabsdiff_f64": (ctypes.c_double, [P, P]),
            "orc_jacobi_solve_f64": (ctypes.c_int, [P, P, ctypes.c_int64, ctypes.c_int64, ctypes.c_double,
                                                    ctypes.c_double, ctypes.POINTER(ctypes.c_int64),
                                                    ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int32)]),
            "orc_vecmat_f64": (ctypes.c_int, [P, P, P, P]),
            "orc_set_threads": (ctypes.c_int, [ctypes.c_int]),
            "orc_pw_advection_f64": (ctypes.c_int, [P, P, P, P, P, P, ctypes.c_void_p, ctypes.c_void_p,
                                                    ctypes.c_void_p, ctypes.c_void_p, ctypes.c_double,
                                                    ctypes.c_double]),
            "orc_tra_adv_f64": (ctypes.c_int, [P, P, P, P, P, P, P, P, P, P, P, ctypes.c_void_p, ctypes.c_int64]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


class OracleError(RuntimeError):
    def __init__(self, code: int, what: str):
        super().__init__(f"oracle {what} failed with code {code}")
        self.code = code


class FArray:
    """A Fortran array view for the oracle: a numpy view + lbounds.

    ``arr`` may be any numpy view (Fortran-ordered whole array, strided or
    negatively strided slice); its byte strides become the descriptor's sm.
    A 0-d array is a scalar operand.
    """

    def __init__(self, arr: np.ndarray, lbounds=None, _desc=None, _owner=None):
        self.arr = arr
        self.owner = _owner if _owner is not None else arr
        if _desc is not None:
            self.desc = _desc
            return
        if arr.dtype not in _NP2TYPE:
            raise TypeError(f"unsupported dtype {arr.dtype}")
        r = arr.ndim
        if r > 3:
            raise ValueError("rank > 3")
        lb = list(lbounds) if lbounds is not None else [1] * r
        d = _Array()
        d.base = arr.ctypes.data
        d.type = _NP2TYPE[arr.dtype]
        d.rank = r
        for k in range(r):
            d.dim[k].lb = lb[k]
            d.dim[k].ext = arr.shape[k]
            d.dim[k].sm = arr.strides[k]
        self.desc = d

    @property
    def rank(self):
        return self.desc.rank

    @property
    def lbounds(self):
        return [self.desc.dim[k].lb for k in range(self.rank)]

    @property
    def shape(self):
        return tuple(self.desc.dim[k].ext for k in range(self.rank))

    @property
    def strides(self):
        return tuple(self.desc.dim[k].sm for k in range(self.rank))

    def base_offset(self) -> int:
        """Byte offset of the first element from the owner's data pointer."""
        return self.desc.base - self.owner.ctypes.data

    def ref(self):
        return ctypes.byref(self.desc)

    def section(self, *triplets) -> "FArray":
        """x(lo:hi:step, ...) with Fortran subscripts (inclusive hi)."""
        r = self.rank
        lo = (ctypes.c_int64 * r)(*[t[0] for t in triplets])
        hi = (ctypes.c_int64 * r)(*[t[1] for t in triplets])
        st = (ctypes.c_int64 * r)(*[t[2] if len(t) > 2 else 1 for t in triplets])
        out = _Array()
        rc = lib().orc_section(self.ref(), lo, hi, st, ctypes.byref(out))
        if rc:
            raise OracleError(rc, "section")
        return FArray(self.arr, _desc=out, _owner=self.owner)

    def view(self) -> np.ndarray:
        """A numpy view of the described elements (shares memory with the owner)."""
        owner = self.owner
        if not (owner.flags.c_contiguous or owner.flags.f_contiguous):
            raise ValueError("owner must be a whole (contiguous) array")
        raw = owner.reshape(-1, order="A").view(np.uint8)
        return np.ndarray(self.shape, dtype=owner.dtype, buffer=raw, offset=self.base_offset(),
                          strides=self.strides)

    def to_numpy(self) -> np.ndarray:
        """Copy out the elements as a plain Fortran-ordered array."""
        return np.array(self.view(), order="F", copy=True)


def _check(rc, what):
    if rc:
        raise OracleError(rc, what)


def triplet_indices(lo: int, hi: int, step: int) -> list[int]:
    n = lib().orc_triplet_indices(lo, hi, step, None, 0)
    if n < 0:
        raise OracleError(n, "triplet")
    buf = (ctypes.c_int64 * max(n, 1))()
    lib().orc_triplet_indices(lo, hi, step, buf, n)
    return list(buf[:n])


def element_offset(a: FArray, *subscripts) -> int:
    j = (ctypes.c_int64 * max(a.rank, 1))(*subscripts)
    return lib().orc_element_offset(a.ref(), j)


def elemental(op: int, dst: FArray, a: FArray, b: FArray, c: FArray | None = None, contract=False):
    _check(lib().orc_elemental(op, dst.ref(), a.ref(), b.ref(), (c or a).ref(), int(contract)), "elemental")


def assign(dst: FArray, src: FArray):
    _check(lib().orc_assign(dst.ref(), src.ref()), "assign")


def sum_seq(x: FArray) -> float:
    return lib().orc_sum_seq_f64(x.ref())


def sum_int(x: FArray) -> int:
    return lib().orc_sum_i32(x.ref()) if x.desc.type == I32 else lib().orc_sum_i64(x.ref())


def sum_exact(x: FArray) -> float:
    return lib().orc_sum_exact_f64(x.ref())


def sum_abs(x: FArray) -> float:
    return lib().orc_sum_abs_f64(x.ref())


def fsum(values) -> float:
    v = np.ascontiguousarray(values, dtype=np.float64)
    return lib().orc_fsum(v.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), v.size)


def tree_combine(values, kind=SUM) -> float:
    v = np.ascontiguousarray(values, dtype=np.float64)
    return lib().orc_tree_combine(v.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), v.size, kind)


def orderR_partials(values, kind=SUM) -> np.ndarray:
    v = np.ascontiguousarray(values, dtype=np.float64)
    nc = (v.size + R_CHUNK - 1) // R_CHUNK
    out = np.empty(max(nc, 1), dtype=np.float64)
    lib().orc_orderR_partials(v.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), v.size, kind,
                              out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    return out[:nc]


def reduce_orderR(x: FArray, kind=SUM) -> float:
    return lib().orc_reduce_orderR_f64(x.ref(), kind)


def maxval(x: FArray):
    if x.desc.type == F64:
        return lib().orc_maxval_f64(x.ref())
    return lib().orc_maxval_int(x.ref())


def minval(x: FArray):
    if x.desc.type == F64:
        return lib().orc_minval_f64(x.ref())
    return lib().orc_minval_int(x.ref())


def dot_products(x: FArray, y: FArray) -> np.ndarray:
    out = np.empty(max(x.shape[0], 1), dtype=np.float64)
    _check(lib().orc_dot_products_f64(x.ref(), y.ref(), out.ctypes.data_as(ctypes.POINTER(ctypes.c_double))),
           "dot_products")
    return out[: x.shape[0]]


def dot_exact(x: FArray, y: FArray) -> tuple[float, float]:
    e = ctypes.c_double()
    a = ctypes.c_double()
    _check(lib().orc_dot_exact_f64(x.ref(), y.ref(), ctypes.byref(e), ctypes.byref(a)), "dot_exact")
    return e.value, a.value


def dot_orderR(x: FArray, y: FArray) -> float:
    p = dot_products(x, y)
    return tree_combine(orderR_partials(p, SUM), SUM)


def transpose(dst: FArray, src: FArray):
    _check(lib().orc_transpose(dst.ref(), src.ref()), "transpose")


def matmul(c: FArray, a: FArray, b: FArray, absum: FArray | None = None):
    _check(lib().orc_matmul_f64(c.ref(), a.ref(), b.ref(), absum.ref() if absum is not None else None),
           "matmul")


def matmul_element(a: FArray, b: FArray, i: int, j: int) -> tuple[float, float]:
    """c(i+1, j+1) (0-based positions) and its sum |a||b|, same order as matmul."""
    t = ctypes.c_double()
    v = lib().orc_matmul_element_f64(a.ref(), b.ref(), i, j, ctypes.byref(t))
    return v, t.value


def set_threads(n: int) -> int:
    """OpenMP threads of the oracle's parallel loops (timing only; results do not depend on it)."""
    return lib().orc_set_threads(n)


def jacobi(u: FArray, unew: FArray, sweeps: int, coeff: float) -> bool:
    r = ctypes.c_int32()
    _check(lib().orc_jacobi_f64(u.ref(), unew.ref(), sweeps, coeff, ctypes.byref(r)), "jacobi")
    return bool(r.value)


JACOBI_C2 = 0.25
JACOBI_C3 = 1.0 / 6.0  # fl(1/6) = 0x1.5555555555555p-3 (R#23)


def product_seq(x: FArray) -> float:
    return lib().orc_product_seq_f64(x.ref())


def product_int(x: FArray) -> int:
    return lib().orc_product_int(x.ref())


def reduce_dim(x: FArray, dim: int, kind: int) -> np.ndarray:
    """SUM/MAXVAL/MINVAL/PRODUCT(x, DIM=dim) as a new Fortran-ordered array (0-d for rank 1)."""
    shape = tuple(e for d, e in enumerate(x.shape) if d != dim - 1)
    out = np.zeros(shape, dtype=x.owner.dtype, order="F")
    _check(lib().orc_reduce_dim(x.ref(), dim, kind, FArray(out).ref()), "reduce_dim")
    return out


def matvec(a: FArray, x: FArray) -> tuple[np.ndarray, np.ndarray]:
    """MATMUL(a(m,k), x(k)) and sum |a(i,l) x(l)| per element."""
    m = a.shape[0]
    y, t = np.zeros(m), np.zeros(m)
    _check(lib().orc_matvec_f64(FArray(y).ref(), a.ref(), x.ref(), FArray(t).ref()), "matvec")
    return y, t


def vecmat(x: FArray, b: FArray) -> tuple[np.ndarray, np.ndarray]:
    """MATMUL(x(k), b(k,n)) and sum |x(l) b(l,j)| per element."""
    n = b.shape[1]
    y, t = np.zeros(n), np.zeros(n)
    _check(lib().orc_vecmat_f64(FArray(y).ref(), x.ref(), b.ref(), FArray(t).ref()), "vecmat")
    return y, t


def maxabsdiff(x: FArray, y: FArray) -> float:
    return lib().orc_maxabsdiff_f64(x.ref(), y.ref())


def jacobi_solve(u: FArray, unew: FArray, max_sweeps: int, check_every: int, tol: float, coeff: float):
    """(sweeps done, last residual, result in unew) -- DESIGN.md R#25."""
    d, r, n = ctypes.c_int64(), ctypes.c_double(), ctypes.c_int32()
    _check(lib().orc_jacobi_solve_f64(u.ref(), unew.ref(), max_sweeps, check_every, tol, coeff, ctypes.byref(d),
                                      ctypes.byref(r), ctypes.byref(n)), "jacobi_solve")
    return d.value, r.value, bool(n.value)


def tra_adv(md: FArray, tsn: FArray, pun: FArray, pvn: FArray, pwn: FArray, umask: FArray, vmask: FArray,
            tmask: FArray, ztfreez: FArray, rnfmsk: FArray, upsmsk: FArray, rnfmsk_z, iters: int) -> None:
    """The tra-adv DO nests (R#28): 3-D fields indexed (ji, jj, jk), the
    2-D fields (ji, jj), rnfmsk_z a float64 vector of length jpk; md is updated in place."""
    nk = md.shape[2]
    z = np.ascontiguousarray(np.asarray(rnfmsk_z, dtype=np.float64))
    if z.shape != (nk,):
        raise ValueError("tra_adv: rnfmsk_z must have length jpk")
    _check(lib().orc_tra_adv_f64(md.ref(), tsn.ref(), pun.ref(), pvn.ref(), pwn.ref(), umask.ref(), vmask.ref(),
                                 tmask.ref(), ztfreez.ref(), rnfmsk.ref(), upsmsk.ref(), ctypes.c_void_p(z.ctypes.data),
                                 iters), "tra_adv")


def pw_advection(su: FArray, sv: FArray, sw: FArray, u: FArray, v: FArray, w: FArray, tzc1, tzc2, tzd1, tzd2,
                 tcx: float, tcy: float) -> None:
    """The pw-advection DO nest (R#26): fields indexed (k, j, i),
    k contiguous; the tz* arrays are float64 vectors of length nz; boundary outputs untouched."""
    nz = u.shape[0]
    zs = [np.ascontiguousarray(np.asarray(z, dtype=np.float64)) for z in (tzc1, tzc2, tzd1, tzd2)]
    for z in zs:
        if z.shape != (nz,):
            raise ValueError("pw_advection: coefficient arrays must have length nz")
    _check(lib().orc_pw_advection_f64(su.ref(), sv.ref(), sw.ref(), u.ref(), v.ref(), w.ref(),
                                      *[ctypes.c_void_p(z.ctypes.data) for z in zs], tcx, tcy), "pw_advection")
