# Profile every configuration's dominant kernel once (ncu --set full) and the headline launch list; run on the GPU box:
#   gpurun -- bash tools/prof_all.sh   (outputs in gpurun_out/, then: python tools/traffic_from_ncu.py gpurun_out/r2_*.ncu-rep)
set -e
cd $GRAFT_REPO_ROOT
for cfg in cfg2 cfg1 cfg3 cfg4 cfg5 cfg2dct; do python tools/prof.py --config $cfg --reps 2; done
python tools/two_sided_prof.py
python bench.py --steps 2 --warmup 3 --others "" --no-cpu --no-sharded > gpurun_out/r2_plain.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches_cfg2.csv python bench.py --steps 2 --warmup 3 --others "" --no-cpu --no-sharded > gpurun_out/r2_ncu_launch.log 2>&1
F="--set full --clock-control none --import-source on -c 1"
ncu $F -k regex:srtt_wht_tc -s 1 -o gpurun_out/r2_cfg2 python tools/prof.py --config cfg2 --reps 3 > /dev/null 2>&1
ncu $F -k regex:sparse_right_cols -s 1 -o gpurun_out/r2_cfg1 python tools/prof.py --config cfg1 --reps 3 > /dev/null 2>&1
ncu $F -k regex:dense_tc_pair -s 1 -o gpurun_out/r2_cfg3 python tools/prof.py --config cfg3 --reps 3 > /dev/null 2>&1
ncu $F -k regex:sparse_adjoint_gather -s 1 -o gpurun_out/r2_cfg4 python tools/prof.py --config cfg4 --reps 3 > /dev/null 2>&1
ncu $F -k regex:dense_tc_pair -s 1 -o gpurun_out/r2_cfg5 python tools/prof.py --config cfg5 --reps 3 > /dev/null 2>&1
ncu $F -k regex:dense_tc_pair -s 1 -o gpurun_out/r2_cfg2dct python tools/prof.py --config cfg2dct --reps 3 > /dev/null 2>&1
ncu $F -k regex:two_sided_kernel -s 1 -o gpurun_out/r2_twosided python tools/two_sided_prof.py > /dev/null 2>&1
ncu $F -k regex:dense_tc_pair -s 1 -o gpurun_out/r2_gauss python tools/prof.py --config gauss --reps 3 > /dev/null 2>&1
echo all-done
