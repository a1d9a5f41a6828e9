"""Reference outputs for BASELINE configs 2 and 3 at full size (512^2), from the REFERENCE itself.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_512.py

Runs the reference's own ``denoise`` (Appendix B of SURVEY.md) on the synthetic counts of
``paper_1609_05722_b200.synth.make_counts`` and stores the denoised image (fp32: the parity gates are
1e-3 * peak) and the full trace (F, G, L,
step_norm, slack, slack_tol) per case.  ~2 minutes of CPU; the GPU box uses the committed npz.
"""

from __future__ import annotations

import dataclasses
import hashlib
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from foepoisson import fileio, pipeline, solver  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
from paper_1609_05722_b200.synth import make_counts  # noqa: E402

CASES = {
    # name: (peak, model, variant, force_branch)
    "cfg2_quad": (1.0, "foe_a", "transform", "quadratic"),
    "cfg2_idiv": (1.0, "foe_a", "transform", None),
    "cfg3_fa": (8.0, "foe_a_original", "direct", None),
    "cfg3_fs": (8.0, "foe_s", "direct", None),
}


def main():
    foe_a = fileio.load_packaged_model("foe_a")
    models = {"foe_a": foe_a, "foe_s": fileio.load_packaged_model("foe_s"),
              "foe_a_original": dataclasses.replace(foe_a, domain_tag="original")}
    out = {}
    for name, (peak, mk, variant, fb) in CASES.items():
        _, y = make_counts(512, 512, 0, peak)
        req = pipeline.DenoiseRequest(noisy=y, peak=peak, model=models[mk], variant=variant, force_branch=fb)
        r = pipeline.denoise(req, solver.SolverConfig(rel_tol=0.0))
        tr = r.trace
        out[f"{name}_image"] = r.image.astype(np.float32)
        out[f"{name}_trace"] = np.array([tr.F, tr.G, tr.L, tr.step_norm, tr.descent_slack, tr.slack_tol]).T
        out[f"{name}_counts_sha"] = np.frombuffer(hashlib.sha256(y.tobytes()).digest(), dtype=np.uint8)
        out[f"{name}_meta"] = np.array([peak, r.lam])
        out[f"{name}_branch"] = np.array(r.branch)
        print(name, r.branch, r.lam, len(tr), flush=True)
    np.savez_compressed(os.path.join(HERE, "cfg23_512.npz"), **out)


if __name__ == "__main__":
    main()
