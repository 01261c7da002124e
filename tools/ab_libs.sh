# A/B of alternative builds of libdppx_gpu.so under _ab/<tag>/ (DPPX_LIB override)
for r in 1 2; do for v in "$@"; do echo "$v $(DPPX_LIB=_ab/$v/libdppx_gpu.so python tools/k1_case.py --b 4 --n 1 --launches 6 2>&1 | tail -1)"; done; done
