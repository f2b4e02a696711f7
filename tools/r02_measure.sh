# Round-2 measurement pass: every profiles/r02_* artefact in one GPU call
# (outputs under gpurun_out/r02_*; copied into profiles/ afterwards).
set -x
python -m paper_2506_02267_b200.build
python -m paper_2506_02267_b200.build --debug
python bench.py > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r02_bench_reference.json 2>&1
python bench.py --config c3 --no-cpu-baseline > gpurun_out/r02_c3.json 2>&1
python bench.py --config c4 --no-cpu-baseline > gpurun_out/r02_c4.json 2>&1
python bench.py --mode fp32 --no-cpu-baseline > gpurun_out/r02_fp32.json 2>&1
timeout 600 python tools/sweep.py > gpurun_out/r02_sweep.jsonl 2> gpurun_out/r02_sweep.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 90 --csv --log-file gpurun_out/r02_launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"skut_tc3|nn_|prep|head" -s 21 -c 7 -o gpurun_out/r02_full python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02_ncu.log 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --cache-control none --clock-control none -k regex:"skut_tc3|nn_|prep|head" -s 21 -c 7 --csv --log-file gpurun_out/r02_dram_warm.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"skut_tc4|nn_select" -s 10 -c 2 -o gpurun_out/r02_tc4 python tools/long_s_run.py 256 bf16 8 > gpurun_out/r02_tc4_ncu.log 2>&1
TAV2_DEBUG=1 timeout 200 python tools/skut_phases.py > gpurun_out/r02_phases.txt 2>&1
TAV2_DEBUG=1 timeout 200 python tools/cta_timeline.py --detail --flush > gpurun_out/r02_cta.txt 2>&1
timeout 300 python tools/overlap_probe.py > gpurun_out/r02_overlap_probe.txt 2>&1
{
  echo "# compute-sanitizer, B200, round 2: smoke() (both modes) and tools/san_c2.py (C2 size, fused twice)"
  for t in memcheck racecheck synccheck; do
    echo "## $t smoke"; timeout 900 compute-sanitizer --tool $t --print-limit 20 python -c 'import __graft_entry__ as g; g.smoke()' 2>&1 | tail -4
    echo "## $t C2"; timeout 1200 compute-sanitizer --tool $t --print-limit 20 python tools/san_c2.py 2>&1 | tail -3
  done
} > gpurun_out/r02_sanitizer.txt 2>&1
ls -la gpurun_out/
