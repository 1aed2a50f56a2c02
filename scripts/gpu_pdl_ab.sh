set -x
python -m pytest tests/test_gpu_kernels.py tests/test_gpu_machinery.py -x -q 2>&1 | tail -3
for i in 1 2; do
TB_STEP_PDL=0 python bench.py --no-kernels > gpurun_out/pdl0_$i.json 2>gpurun_out/pdl0_$i.err
python bench.py --no-kernels > gpurun_out/pdl1_$i.json 2>gpurun_out/pdl1_$i.err
done
for f in gpurun_out/pdl*.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['ms_per_step'], d['roofline']['frac'], d['l2_flushed_per_step']['ms_per_step'], d['clocks'], d['e2e']['value'])"; done
