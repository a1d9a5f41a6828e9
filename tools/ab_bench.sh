#!/bin/bash
# A/B the default library against variant builds on the headline bench (under gpurun).
# usage: bash tools/ab_bench.sh <rounds> <variant.so> [<variant.so> ...]
n=${1:-2}; shift
summ='import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],3),"ms pass",round(d["roofline"]["pass_ms"]*1e3,2),"us e2e",round(d["e2e"]["ms_per_denoise"],3),"trials",d["trials_per_step"],"| 48x7x7",round(d["fallback_48x7"]["ms_per_denoise"],3),"ms pass",round(d["fallback_48x7"]["pass_ms"]*1e3,2),"us")'
for r in $(seq $n); do
  echo -n "default: "; python bench.py --steps 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "$summ"
  for v in "$@"; do
    echo -n "$(basename $v): "; FOE_LIB=$v python bench.py --steps 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "$summ"
  done
done
