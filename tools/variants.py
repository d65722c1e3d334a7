"""Build tuning variants of libftn: one translation unit recompiled with extra -D flags,
linked with the in-tree objects of the others, written to vtmp/libftn_<name>.so.  Load one
with FTN_LIBFTN=vtmp/libftn_<name>.so (paper_2409_18824_b200/ftn.py).

    python tools/variants.py <unit> <name>=<-Dflags ...> [<name>=...]
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2409_18824_b200 import build as B  # noqa: E402


def main():
    unit = sys.argv[1]
    B.build()
    os.makedirs(os.path.join(ROOT, "vtmp"), exist_ok=True)
    objs = [os.path.join(B.BUILD, n + ".o") for n in B.SOURCES if n != unit]
    for spec in sys.argv[2:]:
        name, flags = spec.split("=", 1)
        obj = os.path.join(ROOT, "vtmp", f"{unit}_{name}.o")
        cmd = [B.nvcc()] + B.flags() + flags.split() + ["-Xptxas", "-v", "-c", os.path.join(B.CSRC, unit + ".cu"), "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode:
            sys.exit(r.stderr[-3000:])
        open(os.path.join(ROOT, "vtmp", f"{unit}_{name}.ptxas.log"), "w").write(r.stderr)
        lib = os.path.join(ROOT, "vtmp", f"libftn_{name}.so")
        nccl_lib = os.path.join(B.nccl_root(), "lib")
        cmd = [B.nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", lib] + objs + [obj] + [
            "-L" + nccl_lib, "-l:libnccl.so.2", "-Xlinker", "-rpath," + nccl_lib, "-cudart", "static"]
        subprocess.run(cmd, check=True)
        print("built", lib)


if __name__ == "__main__":
    main()
