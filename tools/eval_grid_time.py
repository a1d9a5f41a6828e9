"""Wall time of the reference-sized evaluation grid on the device (8 images 256^2 x 7 peaks x 2 variants)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1609_05722_b200 as fp  # noqa: E402
from paper_1609_05722_b200 import evaluate as ev  # noqa: E402

spec = ev.BenchmarkSpec(images=tuple(f"syn256x256s{i}" for i in range(8)), peaks=(0.1, 0.2, 0.5, 1.0, 2.0, 4.0, 40.0),
                        variants=("transform", "transform_binned"), transform_model=fp.load_packaged_model("foe_a"))
ev.run_benchmark(ev.BenchmarkSpec(images=("syn64x64s0",), peaks=(1.0,), variants=spec.variants,
                                  transform_model=spec.transform_model))  # warm-up
t0 = time.perf_counter()
rows = ev.run_benchmark(spec)
dt = time.perf_counter() - t0
print(f"{len(rows)} jobs in {dt:.2f} s ({dt / len(rows) * 1e3:.1f} ms/job)")
for r in ev.average_rows(rows):
    print(f"  avg peak {r.peak:5g} {r.variant:17s} PSNR {r.psnr_db:7.3f} MSSIM {r.mssim:.4f}")
