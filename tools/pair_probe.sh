#!/bin/bash
# CTA-pair dense engine (cta_group::2) vs the single-CTA engine at configs 3 and 5
run() { env "$@" python bench.py --config $CFG --others "" --no-cpu --no-sharded --steps 10 --warmup 3 2>>gpurun_out/pair_err.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$CFG $*', round(d['ms_per_step'],4), round(d['roofline']['frac'],3))"; }
for CFG in cfg5 cfg3; do
  run SKETCH_B200_TC_PAIR=0
  run SKETCH_B200_TC_PAIR=1
done
