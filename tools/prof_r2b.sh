# Re-capture the kernels changed in the second half of round 2 (K1c for config 1, K4 sign-bit weights +
# lockstep for config 5) and the headline bench line; run on the GPU box:
#   gpurun -- bash tools/prof_r2b.sh   (then: python tools/traffic_from_ncu.py gpurun_out/r2_cfg1.ncu-rep gpurun_out/r2_cfg5.ncu-rep)
cd $GRAFT_REPO_ROOT
python bench.py > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err
F="--set full --clock-control none --import-source on -c 1"
ncu $F -k regex:sparse_right_cols -s 1 -o gpurun_out/r2_cfg1 python tools/prof.py --config cfg1 --reps 3 > gpurun_out/ncu_cfg1.log 2>&1
ncu $F -k regex:dense_tc_pair -s 1 -o gpurun_out/r2_cfg5 python tools/prof.py --config cfg5 --reps 3 > gpurun_out/ncu_cfg5.log 2>&1
echo all-done
