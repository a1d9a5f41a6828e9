"""Build the timing-diagnostic variant of the CUDA library (per-block cycle stamps of the tensor-core pass).

usage: python tools/build_diag.py  ->  paper_1609_05722_b200/libfoe_b200_stamps.so
then:  FOE_LIB=paper_1609_05722_b200/libfoe_b200_stamps.so python tools/diag_times.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1609_05722_b200 import _lib  # noqa: E402

if __name__ == "__main__":
    print(_lib.build(force=True, out=os.path.join(_lib.PKG, "libfoe_b200_stamps.so"), defines=("FOE_STAMPS=1",)))
