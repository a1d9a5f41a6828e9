#!/bin/bash
# Quick GPU check of a kernel change: operator / gradient parity tests, then the headline bench line.
# usage (under gpurun): bash tools/gpu_quick.sh <tag> [pytest -k expression]
tag=${1:-q}
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q ${2:+-k "$2"} > gpurun_out/quick_tests_$tag.log 2>&1
tail -3 gpurun_out/quick_tests_$tag.log
grep -E "^E  " gpurun_out/quick_tests_$tag.log | head -8
timeout 120 python bench.py --steps 10 --no-cpu-baseline > gpurun_out/quick_bench_$tag.log 2>&1
tail -1 gpurun_out/quick_bench_$tag.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value',round(d['value'],1),'ms',round(d['ms_per_step'],3),'pass_us',round(d['roofline']['pass_ms']*1e3,2),'frac',round(d['roofline']['frac'],4),'e2e_ms',round(d['e2e']['ms_per_denoise'],3), 'trials', d['trials_per_step'], '48x7', round(d['fallback_48x7']['ms_per_denoise'],3))"
