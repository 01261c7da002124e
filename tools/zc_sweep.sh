set -x
python -m pytest tests/test_gpu_parity.py -q -x -k "small_frame_paths or single_frame_graph or pageable" 2>&1 | tail -5
for u in 4096 8192 12288 16384; do for c in 0 12 18 36; do echo "unit=$u ctas=$c"; DPPX_ZC_UNIT=$u DPPX_ZC_CTAS=$c python tools/latency_probe.py | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['median_us'], d['p10_us'], d['kernel_us_per_call'])"; done; done
DPPX_ZEROCOPY=0 python tools/latency_probe.py
python tools/latency_probe.py 576 768 3 16 a
