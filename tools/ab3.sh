# A/B (_ab/old vs _ab/new): headline bench K1 + draw-bound K1 cases
for r in 1 2; do for v in old new; do
  echo "$v headline $(DPPX_LIB=_ab/$v/libdppx_gpu.so python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d["roofline"]; print(d["value"], r["avg_launch_ms"], r["frac"])')"
  for c in "--b 16 --n 4 --complex 0.5" "--b 16 --n 4 --complex 0.25" "--b 16 --n 4 --complex 0.9" "--b 8 --n 2 --complex 0.5" "--b 32 --n 8 --complex 0.5"; do
    echo "$v $c $(DPPX_LIB=_ab/$v/libdppx_gpu.so python tools/k1_case.py $c --launches 6 2>&1 | tail -1)"; done
done; done
