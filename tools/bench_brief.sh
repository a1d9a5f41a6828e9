#!/bin/bash
# one-line bench summary: value, ms per step, pass us, trials (extra args go to bench.py)
python bench.py --steps 5 --no-cpu-baseline "$@" 2>/dev/null | tail -1 | python3 -c "
import json,sys
d=json.loads(sys.stdin.read())
print('value',round(d['value'],1),'ms',round(d['ms_per_step'],3),'pass_us',round(d['roofline']['pass_ms']*1e3,2),'trials',d['trials_per_step'])"
