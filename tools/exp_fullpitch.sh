#!/bin/bash
# A/B of dppx_ctx_set_out_pad_scratch (run under gpurun): GPU tests, the
# padded-row bench shapes with and without it, the headline, the fuzz.
TAG=${1:-r01m}
OUT=gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > $OUT/pytest_gpu_$TAG.log 2>&1
echo "pytest_rc=$?"; tail -2 $OUT/pytest_gpu_$TAG.log
for w in celeba sweep; do
  timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline > $OUT/bench_${w}_$TAG.log 2>&1; echo "${w}=$?"
  timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-pad-scratch > $OUT/bench_${w}_nopad_$TAG.log 2>&1; echo "${w}_nopad=$?"
done
timeout 600 python bench.py > $OUT/bench_$TAG.log 2>&1; echo "bench_rc=$?"
timeout 900 python tools/fuzz_gpu.py --cases 1500 --seed 23 > $OUT/fuzz_$TAG.txt 2>&1; echo "fuzz_rc=$?"; tail -1 $OUT/fuzz_$TAG.txt
for f in $OUT/bench_*$TAG.log; do echo $f; tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['frac'], d.get('reconstruct'), (d.get('e2e') or {}).get('value'))" 2>&1 | tail -1; done
