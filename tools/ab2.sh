bash tools/ab_bench.sh celeba 4k
for v in old new; do for c in "--b 4 --n 1" "--b 16 --n 4 --complex 0.5"; do echo "$v $c $(DPPX_LIB=_ab/$v/libdppx_gpu.so python tools/k1_case.py $c --launches 6 2>&1 | tail -1)"; done; done
