bash tools/ab_bench.sh h37 h24 h18
