#!/bin/bash
# One gpurun call: tests, smoke, bench variants, PCIe probe, ablation cells, ncu.
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
python scripts/pcie_probe.py > gpurun_out/pcie.json 2>&1; cat gpurun_out/pcie.json
for impl in reg regpf bulk; do
  timeout 600 python bench.py --steps 200 --warmup 10 --no-cpu-baseline --step-impl $impl --e2e-steps 5 > gpurun_out/bench_$impl.json 2>&1; tail -c 1200 gpurun_out/bench_$impl.json
done
for impl in reg regpf bulk; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_step -s 18 -c 1 -o gpurun_out/prof_k2_$impl python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline --step-impl $impl > gpurun_out/ncu_full_$impl.log 2>&1
done
timeout 900 python -m paper_2303_08058_b200.cli --subgrids 512 --steps 5 --repeats 1 --workers 8 --executors 32 --max-agg 8 --output json > gpurun_out/ablation_512.json 2> gpurun_out/ablation_512.err; cat gpurun_out/ablation_512.json | head -40; tail -5 gpurun_out/ablation_512.err
ls -la gpurun_out
