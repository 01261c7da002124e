# A/B of two builds (_ab/old, _ab/new) on bench workloads: K1 ms per launch
for r in 1 2; do for v in old new; do for w in "$@"; do
  echo "$v $w $(DPPX_LIB=_ab/$v/libdppx_gpu.so python bench.py --workload $w --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d["roofline"]; print(d["value"], r["avg_launch_ms"], r["frac"])')"
done; done; done
