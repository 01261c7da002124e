#!/bin/bash
# Round-2 evidence on one B200 (run under gpurun): tests, smoke, every bench
# workload, the reference arm, ncu launch list + full capture of the headline
# step, the reference's own gate / unit suites on the drop-in, latency, sweeps,
# the multi-rank launch. Outputs: gpurun_out/<TAG>_*
TAG=${1:-r02x}
O=gpurun_out/$TAG
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,memory.total --format=csv > ${O}_box.txt
lscpu | grep -E "Model name|^CPU\(s\)" >> ${O}_box.txt
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > ${O}_pytest_gpu.txt 2>&1
echo "pytest_rc=$?"; tail -2 ${O}_pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > ${O}_smoke.txt 2>&1; echo "smoke_rc=$?"; tail -1 ${O}_smoke.txt
timeout 900 python bench.py > ${O}_bench.json 2> ${O}_bench.err; echo "bench_rc=$?"
timeout 900 python bench.py --impl reference > ${O}_bench_reference.json 2>&1; echo "bench_ref_rc=$?"
for w in pets pets_clip 4k celeba sweep; do
  timeout 900 python bench.py --workload $w --no-cpu-baseline > ${O}_bench_$w.json 2> ${O}_bench_$w.err; echo "bench_${w}_rc=$?"
done
DPPX_DIST_BACKEND=gloo DPPX_FORCE_DEVICE=0 timeout 900 python bench.py --gpus 2 --frames 300 --no-cpu-baseline \
    > ${O}_bench_gpus2_gloo_onegpu.json 2> ${O}_bench_gpus2.err; echo "bench_gpus2_rc=$?"
B="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
$B > /dev/null 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file ${O}_launches.csv $B > /dev/null 2>&1; echo "ncu_launch_rc=$?"
B1="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_stats_tma|k_classify" -s 2 -c 2 \
    -o ${O}_k0_k1_full $B1 > /dev/null 2>&1; echo "ncu_full_rc=$?"
./tests/cpp/_ref_gate/dppix_acceptance_gpu > ${O}_reference_gate_on_dropin.txt 2>&1; echo "gate_rc=$?"
./tests/cpp/_ref_gate/dppix_unit_gpu > ${O}_reference_unit_suites_on_dropin.txt 2>&1; echo "unit_rc=$?"
python tools/latency_probe.py > ${O}_latency.txt 2>&1                       # default: K1z zero-copy
DPPX_ZEROCOPY=0 python tools/latency_probe.py >> ${O}_latency.txt 2>&1      # CUDA graph
DPPX_ZEROCOPY=0 DPPX_GRAPH=0 python tools/latency_probe.py >> ${O}_latency.txt 2>&1  # staged
python tools/latency_probe.py 576 768 3 16 a >> ${O}_latency.txt 2>&1
DPPX_ZEROCOPY=1 python tools/latency_probe.py 576 768 3 16 a >> ${O}_latency.txt 2>&1
[ -x tools/pcie_probe ] || nvcc -O2 -gencode arch=compute_100a,code=sm_100a -o tools/pcie_probe tools/pcie_probe.cu
./tools/pcie_probe > ${O}_pcie_probe.txt 2>&1
for c in "--b 4 --n 1" "--b 4 --n 1 --eps 0.1" "--b 16 --n 4 --complex 0.5" "--b 16 --n 4"; do
  echo "$c $(python tools/k1_case.py $c --launches 6 2>&1 | tail -1)" >> ${O}_k1_cases.txt; done
timeout 900 python tools/b_sweep.py 120 > ${O}_b_sweep.json 2>/dev/null
timeout 900 python tools/b_sweep.py 120 uniform > ${O}_b_sweep_uniform.json 2>/dev/null
timeout 900 python tools/k1_complex_sweep.py > ${O}_k1_complex_sweep.json 2>/dev/null
timeout 900 python tools/batch_bench.py > ${O}_batch.json 2>/dev/null; echo "batch_rc=$?"
echo done
