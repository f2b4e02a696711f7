# Measurement pass: every profiles/ artefact in one GPU call (outputs under gpurun_out/r02_*).
set -x
python bench.py > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r02_bench_reference.json 2>&1
python bench.py --config c3 --no-cpu-baseline > gpurun_out/r02_c3.json 2>&1
python bench.py --config c4 --no-cpu-baseline > gpurun_out/r02_c4.json 2>&1
python bench.py --mode fp32 --no-cpu-baseline > gpurun_out/r02_fp32.json 2>&1
python tools/sweep.py > gpurun_out/r02_sweep.jsonl 2> gpurun_out/r02_sweep.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/r02_launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"skut_tc3|nn_|prep" -s 18 -c 6 -o gpurun_out/r02_full python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02_ncu.log 2>&1
# DRAM bytes with the L2 kept warm across kernels (no cache flush between
# the replayed kernels): the traffic a step really causes
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --cache-control none --clock-control none -k regex:"skut_tc3|nn_|prep" -s 18 -c 6 --csv --log-file gpurun_out/r02_dram_warm.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
# the long-layout kernel (k_ll = 256, S = 352: skut_tc4 on 2-CTA clusters)
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"skut_tc4|nn_select" -s 10 -c 2 -o gpurun_out/r02_tc4 python tools/long_s_run.py 256 bf16 8 > gpurun_out/r02_tc4_ncu.log 2>&1
TAV2_DEBUG=1 timeout 200 python tools/skut_phases.py > gpurun_out/r02_phases.txt 2>&1
TAV2_DEBUG=1 timeout 200 python tools/cta_timeline.py --detail --flush > gpurun_out/r02_cta.txt 2>&1
timeout 300 python tools/overlap_probe.py > gpurun_out/r02_overlap_probe.txt 2>&1
ls -la gpurun_out/
