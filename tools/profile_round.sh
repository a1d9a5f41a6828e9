#!/bin/bash
# Round-end evidence on the GPU box: default bench line, launch list of a short bench run, one ncu --set full
# capture of the trial pass on the converged config-2 state (the 211th k_pass_tc launch of a 1-step bench:
# 208 solve launches -- INIT, 206 trials, final energy -- then the back-to-back bench passes).
# usage (under gpurun): bash tools/profile_round.sh <tag>
tag=${1:-final}
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
tail -1 gpurun_out/bench_$tag.json
cmd="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --pass-reps 5"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$tag.csv $cmd \
  > gpurun_out/launches_$tag.log 2>&1
echo "launch list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_pass_tc -s 210 -c 1 -o gpurun_out/prof_$tag \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-fallback --pass-reps 2 > gpurun_out/ncu_$tag.log 2>&1
echo "ncu rc=$?"
