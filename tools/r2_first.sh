set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -o /tmp/mma_bench tools/mma_bench.cu -lcuda && timeout 60 /tmp/mma_bench > gpurun_out/mma_bench.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.txt 2>&1; echo rc=$?
timeout 300 python bench.py > gpurun_out/bench.txt 2>&1
tail -3 gpurun_out/gputest.txt; cat gpurun_out/mma_bench.txt; tail -1 gpurun_out/bench.txt | cut -c1-600
