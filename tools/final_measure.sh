# Round-end measurement pass: every profiles/ artefact in one GPU call (outputs under gpurun_out/f_*).
set -x
python bench.py > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err
python bench.py --config c3 --no-cpu-baseline > gpurun_out/f_c3.json 2>&1
python bench.py --config c4 --no-cpu-baseline > gpurun_out/f_c4.json 2>&1
python bench.py --mode fp32 --no-cpu-baseline > gpurun_out/f_fp32.json 2>&1
python tools/sweep.py > gpurun_out/f_sweep.jsonl 2> gpurun_out/f_sweep.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/f_launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"skut_tc3|nn_|prep" -s 18 -c 6 -o gpurun_out/f_full python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/f_ncu.log 2>&1
TAV2_DEBUG=1 timeout 200 python tools/skut_phases.py > gpurun_out/f_phases.txt 2>&1
TAV2_DEBUG=1 timeout 200 python tools/cta_timeline.py --detail > gpurun_out/f_cta.txt 2>&1
ls -la gpurun_out/
