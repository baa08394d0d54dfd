"""Write tests/golden/fseg_ref_{harm,biharm}_Mt10.bin with the REFERENCE's own
save_mollified_green (greens.cpp:155-171, oracle/_ref): the FSEG cache files the
GPU loader must read and reproduce byte for byte (tests/test_gpu_fseg.py).
Ltilde = 1.25, Mtilde = 10 (D = 20), sf = 1 + sqrt(3): 64 KB each.

    python tests/golden/make_fseg.py
"""
import math
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import refimpl as R  # noqa: E402

if __name__ == "__main__":
    for gk, nm in ((0, "harm"), (1, "biharm")):
        path = os.path.join(HERE, f"fseg_ref_{nm}_Mt10.bin")
        R.save_green(gk, 1.25, 10, 1.0 + math.sqrt(3.0), path)
        print("wrote", path, os.path.getsize(path))
