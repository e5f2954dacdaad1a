#!/bin/bash
# Round-end evidence of the current build, one GPU call: bash scripts/final_evidence.sh  (outputs under gpurun_out/final/)
out=gpurun_out/final; mkdir -p $out
( time python -m pytest tests -m gpu -x -q ) > $out/gputest.log 2>&1
tail -3 $out/gputest.log
for c in c1 c2 c3; do python bench.py --workload $c --steps 10 --warmup 3 > $out/bench_$c.json 2> $out/bench_$c.err; done
python bench.py --workload c5 --steps 5 --warmup 3 > $out/bench_c5.json 2> $out/bench_c5.err
python bench.py --steps 3 --warmup 3 > $out/bench_c4.json 2> $out/bench_c4.err
python bench.py --impl reference --steps 1 --warmup 0 > $out/reference_arm_c4.json 2> $out/reference_arm_c4.err
python bench.py --sharded --steps 3 --warmup 3 > $out/bench_c4_sharded_1rank.json 2> $out/bench_c4_sharded.err
# checked build (device bounds checks) on the suites that touch the changed kernels + sanitizer workloads
( DSCR_LIB=checked python scripts/sanitize_workload.py all; echo rc=$?; DSCR_LIB=checked python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py tests/test_gpu_batched.py tests/test_gpu_c5_bench.py tests/test_gpu_tall.py tests/test_gpu_robustness.py tests/test_gpu_seams.py tests/test_gpu_acceptance.py -q 2>&1 | tail -2; echo rc=$? ) > $out/checked.log 2>&1
# c5: launch list and ncu --set full of the per-iteration kernels (after the plain runs above exited 0)
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $out/c5_launches.csv python scripts/c5_one_solve.py > $out/ncu_c5l.log 2>&1
python scripts/launch_summary.py $out/c5_launches.csv > $out/c5_launch_summary.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_bresid_w|k_bupdate_warp|k_gemm_dt" -s 120 -c 3 -o $out/c5_iter -f python scripts/c5_iteration_profile.py > $out/ncu_c5i.log 2>&1
for c in c1 c2 c3; do timeout 300 python scripts/timing_breakdown.py $c; done > $out/stamps_c1_c3.txt 2>&1
ls -la $out
