# Re-capture the kernels changed in the second half of round 2 and the final bench line; run on the
# GPU box:  gpurun -- bash tools/prof_r2b.sh
# (then: python tools/traffic_from_ncu.py gpurun_out/r2_{cfg1,cfg3,cfg5,cfg2dct,twosided}.ncu-rep)
cd $GRAFT_REPO_ROOT
python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo rc=$? >> gpurun_out/gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
python bench.py > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err
F="--set full --clock-control none --import-source on -c 1"
ncu $F -k regex:sparse_right_cols -s 1 -o gpurun_out/r2_cfg1 python tools/prof.py --config cfg1 --reps 3 > gpurun_out/ncu_cfg1.log 2>&1
ncu $F -k regex:dense_tc_pair -s 1 -o gpurun_out/r2_cfg3 python tools/prof.py --config cfg3 --reps 3 > gpurun_out/ncu_cfg3.log 2>&1
ncu $F -k regex:dense_tc_pair -s 1 -o gpurun_out/r2_cfg5 python tools/prof.py --config cfg5 --reps 3 > gpurun_out/ncu_cfg5.log 2>&1
ncu $F -k regex:dense_tc_pair -s 1 -o gpurun_out/r2_cfg2dct python tools/prof.py --config cfg2dct --reps 3 > gpurun_out/ncu_cfg2dct.log 2>&1
ncu $F -k regex:two_sided_kernel -s 1 -o gpurun_out/r2_twosided python tools/two_sided_prof.py > gpurun_out/ncu_ts.log 2>&1
echo all-done
