#!/bin/bash
# Secondary measurements (run under gpurun): per-shape bench lines, the K1
# complex-fraction sweep, the variance-extension bench.
TAG=${1:-r01}
OUT=gpurun_out
for w in pets 4k celeba sweep; do
  timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline > $OUT/bench_${w}_$TAG.log 2>&1
  echo "bench_${w}_rc=$?"
done
timeout 300 python tools/k1_complex_sweep.py > $OUT/k1_sweep_$TAG.json 2>&1; echo "sweep_rc=$?"
timeout 300 python tools/variance_bench.py --steps 10 > $OUT/variance_$TAG.json 2>&1; echo "var_rc=$?"
timeout 300 python tools/b_sweep.py 120 > $OUT/b_sweep_$TAG.json 2>&1; echo "b_sweep_rc=$?"
timeout 900 python tools/fuzz_gpu.py --cases 1500 --seed 21 > $OUT/fuzz_$TAG.txt 2>&1; echo "fuzz_rc=$?"; tail -1 $OUT/fuzz_$TAG.txt
timeout 300 python tools/b_sweep.py 120 uniform > $OUT/b_sweep_uniform_$TAG.json 2>&1; echo "b_sweep_uniform_rc=$?"
timeout 600 python tools/batch_bench.py --files 64 > $OUT/batch_$TAG.json 2>&1; echo "batch_rc=$?"; tail -1 $OUT/batch_$TAG.json | cut -c1-400
