#!/bin/bash
# One build->measure cycle on the GPU box: parity tests, smoke, bench, one ncu capture of the trial pass.
# usage (under gpurun): bash tools/gpu_cycle.sh <tag> [extra pytest args]
tag=${1:-run}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q ${2:-} > gpurun_out/gpu_tests_$tag.log 2>&1
tail -2 gpurun_out/gpu_tests_$tag.log
grep -E "^E  .*(Assert|\(|Error)" gpurun_out/gpu_tests_$tag.log | head -8
python __graft_entry__.py smoke 2>&1 | tail -1
python bench.py --steps 5 > gpurun_out/bench_$tag.log 2>&1
tail -1 gpurun_out/bench_$tag.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value',round(d['value'],1),'ms',round(d['ms_per_step'],3),'pass_us',round(d['roofline']['pass_ms']*1e3,2),'frac',round(d['roofline']['frac'],4),'e2e',round(d['e2e']['value'],1), 'trials', d['trials_per_step'], 'clk', d['clocks'])"
python bench.py --steps 1 --warmup 0 --no-cpu-baseline --pass-reps 2 > gpurun_out/plain_$tag.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_pass -s 40 -c 1 -o gpurun_out/prof_$tag \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline --pass-reps 2 > gpurun_out/ncu_$tag.log 2>&1
tail -1 gpurun_out/ncu_$tag.log
