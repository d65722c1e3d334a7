"""Time TRANSPOSE through the C ABI: GB/s (2 x elem_len bytes per element) for int32 and real(8).

    python tools/time_transpose.py            (FTN_TRANSPOSE_NO_TMA=1: the LDG/STG path)
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2409_18824_b200 import ftn  # noqa: E402


def main():
    torch.cuda.set_device(0)
    for dtype, n1, n2 in ((torch.int32, 32768, 32768), (torch.float64, 16384, 16384), (torch.int32, 8192, 4096),
                          (torch.float64, 30000, 7000)):
        A = ftn.FArray.empty((n1, n2), dtype=dtype)
        B = ftn.FArray.empty((n2, n1), dtype=dtype)
        A.tensor.random_(0, 1 << 20)
        for _ in range(3):
            ftn.transpose(B, A)
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        reps = 10
        ev[0].record()
        for _ in range(reps):
            ftn.transpose(B, A)
        ev[1].record()
        torch.cuda.synchronize()
        ms = ev[0].elapsed_time(ev[1]) / reps
        nbytes = 2 * n1 * n2 * A.tensor.element_size()
        ok = torch.equal(B.tensor, A.tensor.t())
        print(f"{str(dtype):14s} {n1}x{n2}: {ms:.3f} ms {nbytes / ms / 1e6:.0f} GB/s exact={ok}")
        del A, B
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
