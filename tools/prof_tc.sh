#!/bin/bash
# launch lists + one full ncu capture of the dense engine (configs 3 and 5); run after the plain bench exits 0
for CFG in cfg3 cfg5; do
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$CFG.csv \
      python bench.py --config $CFG --others "" --no-cpu --no-sharded --steps 2 --warmup 3 > /dev/null 2>&1
  ncu --set full --clock-control none --import-source on -k regex:dense_tc -s 2 -c 1 -o gpurun_out/ncu_tc_$CFG \
      python bench.py --config $CFG --others "" --no-cpu --no-sharded --steps 1 --warmup 3 > gpurun_out/ncu_$CFG.log 2>&1
done
