# K1z tuning sweep (unit bytes x CTAs) on the PETS frame; see profiles/r02_zerocopy.txt
for u in 3072 6144 12288; do for c in 0 36 54 72 108; do echo "unit=$u ctas=$c $(DPPX_ZC_UNIT=$u DPPX_ZC_CTAS=$c python tools/latency_probe.py | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['median_us'], d['p10_us'], d['kernel_us_per_call'])")"; done; done
