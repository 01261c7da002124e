python -m pytest tests/test_gpu_parity.py -q -x -k "fast_path or one_read_sweep or lg2 or keyed or ks" 2>&1 | tail -2
for i in 1 2; do
python tools/k1_case.py --b 4 --n 1 --launches 6 2>&1 | tail -1
python tools/k1_case.py --b 4 --n 1 --eps 0.1 --launches 6 2>&1 | tail -1
python tools/k1_case.py --b 16 --n 4 --complex 0.5 --launches 6 2>&1 | tail -1
python tools/k1_case.py --b 16 --n 4 --launches 6 2>&1 | tail -1
done
