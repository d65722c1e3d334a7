"""PCIe probe for the e2e leg of bench.py: pinned host <-> device copy bandwidth of one
512 MiB buffer (the 8192^2 real(8) array), one direction at a time and both at once.
Usage: python tools/pcie_probe.py  -> one JSON line (GB/s)."""
import json

import torch


def main():
    n = 8192 * 8192
    reps = 6
    hs = [torch.empty(n, dtype=torch.float64, pin_memory=True) for _ in range(2)]
    ds = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(2)]
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    res = {}

    def run(name, h2d, d2h):
        for warm in (True, False):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            s1.wait_event(e0)
            s2.wait_event(e0)
            for _ in range(1 if warm else reps):
                if h2d:
                    with torch.cuda.stream(s1):
                        ds[0].copy_(hs[0], non_blocking=True)
                if d2h:
                    with torch.cuda.stream(s2):
                        hs[1].copy_(ds[1], non_blocking=True)
            for st in (s1, s2):
                ev = torch.cuda.Event()
                ev.record(st)
                torch.cuda.current_stream().wait_event(ev)
            e1.record()
            torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        res[name] = round(n * 8 * (int(h2d) + int(d2h)) / ms / 1e6, 1)
        res[name + "_ms"] = round(ms, 3)

    run("h2d", True, False)
    run("d2h", False, True)
    run("both", True, True)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
