#!/bin/bash
# Round evidence on one B200 (run under gpurun): tests, bench (both arms),
# ncu launch list of the bench command, one ncu --set full capture of K0 + K1.
TAG=${1:-r01}
OUT=gpurun_out
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,memory.total --format=csv > $OUT/gpu_$TAG.txt
lscpu | grep -E "Model name|^CPU\(s\)" >> $OUT/gpu_$TAG.txt
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > $OUT/pytest_gpu_$TAG.log 2>&1
echo "pytest_rc=$?"; tail -2 $OUT/pytest_gpu_$TAG.log
timeout 600 python bench.py > $OUT/bench_$TAG.log 2>&1; echo "bench_rc=$?"
timeout 600 python bench.py --impl reference > $OUT/bench_ref_$TAG.log 2>&1; echo "bench_ref_rc=$?"
B="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
$B > $OUT/plain_$TAG.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv $B > $OUT/ncu_launch_$TAG.log 2>&1
echo "ncu_launch_rc=$?"
B1="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$B1 > $OUT/plain1_$TAG.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_stats_tma|k_classify" -s 2 -c 2 -o $OUT/full_$TAG $B1 > $OUT/ncu_full_$TAG.log 2>&1
echo "ncu_full_rc=$?"
tail -1 $OUT/bench_$TAG.log | cut -c1-600
tail -1 $OUT/bench_ref_$TAG.log | cut -c1-300
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > $OUT/smoke_$TAG.log 2>&1; echo "smoke_rc=$?"; tail -1 $OUT/smoke_$TAG.log
