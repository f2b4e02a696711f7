for g in 0 143 0 143 125; do
  TAV2_SKUT_GRID=$g python bench.py --steps 300 --warmup 20 --no-cpu-baseline > gpurun_out/g.txt 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/g.txt').read().strip().splitlines()[-1]); print('grid $g', d['value'], d['ms_per_step'], d['kernels']['skut_tc3']['ms_per_launch'], d['e2e']['value'])"
done
