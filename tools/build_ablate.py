"""Build the ablation variants of the CUDA library for tools/ablate.sh (timing diagnostics; results are wrong)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1609_05722_b200 import _lib  # noqa: E402

for v in (0, 1, 2, 4, 8, 16, 6, 31):
    print(_lib.build(force=True, out=os.path.join(_lib.PKG, f"libfoe_b200_ab{v}.so"), defines=("FOE_STAMPS=1", f"FOE_ABLATE={v}")))
