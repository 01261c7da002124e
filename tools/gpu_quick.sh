#!/bin/bash
# One gpurun session: GPU tests, a bench line, and an ncu capture of K1.
# usage (under gpurun): bash tools/gpu_quick.sh [tag] [extra bench args]
TAG=${1:-run}; shift
OUT=gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > $OUT/pytest_gpu_$TAG.log 2>&1
echo "pytest_rc=$?"; tail -3 $OUT/pytest_gpu_$TAG.log
timeout 400 python bench.py --steps 5 --warmup 3 --no-e2e "$@" > $OUT/bench_$TAG.log 2>&1
echo "bench_rc=$?"; tail -1 $OUT/bench_$TAG.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value',d['value'],'frac',d['roofline']['frac'],'k1_ms',d['roofline']['avg_launch_ms'],'k0_ms',d['roofline']['k0_ms_per_launch'],'step_frac',d['roofline']['step_frac_incl_K0'])"
B="python bench.py --frames 60 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$B > $OUT/b60_$TAG.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_stats_tma -s 1 -c 1 -o $OUT/prof_$TAG $B > $OUT/ncu_$TAG.log 2>&1
echo "ncu_rc=$?"
