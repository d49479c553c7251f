#!/bin/bash
# quick K1 timing at config 1 (persistent variants vs classic)
run() { env "$@" python bench.py --config cfg1 --others "" --no-cpu --no-sharded --steps 20 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$*', round(d['ms_per_step'],4), round(d['roofline']['frac'],3))"; }
run SKETCH_B200_K1_CLASSIC=0
run SKETCH_B200_K1_NEED=16
run SKETCH_B200_K1_NEED=4
run SKETCH_B200_K1_CLASSIC=0
