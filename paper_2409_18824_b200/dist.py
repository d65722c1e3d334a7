"""Slab decomposition along the last Fortran dimension.

Pure host arithmetic shared by bench.py and the tests; the exchange itself is
ftn_jacobi_dist / ftn_*_global in libftn (NCCL).  In column-major storage a
last-dimension slab is one contiguous block and so is each of its halo planes.
"""
from __future__ import annotations

from dataclasses import dataclass

R_CHUNK = 65536  # DESIGN.md §4.2 step 2


@dataclass(frozen=True)
class Slab:
    rank: int
    nranks: int
    lo: int          # first owned global plane (0-based position in the last dim)
    hi: int          # one past the last owned plane
    halo_lo: bool    # a halo plane precedes the owned planes in the local array
    halo_hi: bool

    @property
    def owned(self) -> int:
        return self.hi - self.lo


def slab(n_last: int, nranks: int, rank: int) -> Slab:
    """Owned planes [lo, hi) of rank `rank` when n_last planes are split as evenly as possible
    (the first n_last % nranks ranks get one extra plane)."""
    if not 0 <= rank < nranks:
        raise ValueError("rank out of range")
    base, extra = divmod(n_last, nranks)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return Slab(rank, nranks, lo, hi, rank > 0, rank < nranks - 1)


def jacobi_slab(n_last: int, nranks: int, rank: int, halo: int = 1) -> tuple[int, int]:
    """Interior planes 1..n_last-2 are split over the ranks; the local array of a rank spans
    its owned planes plus `halo` halo planes on each side (the first / last rank's outermost
    planes beyond the global boundary plane are never consumed).  Returns (first global plane
    of the local array, local extent)."""
    s = slab(n_last - 2, nranks, rank)
    return s.lo + 1 - halo, s.owned + 2 * halo


def reduction_slab_aligned(n_elems: int, plane_elems: int, nranks: int) -> bool:
    """True when every rank's slab is the same power-of-two number of R chunks, which makes
    the distributed fp64 SUM bit-identical to the 1-GPU result (DESIGN.md §4.2 step 7)."""
    if n_elems % nranks:
        return False
    per = n_elems // nranks
    if per % plane_elems or per % R_CHUNK:
        return False
    chunks = per // R_CHUNK
    return chunks & (chunks - 1) == 0
