set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q -k "not fuzz" 2>&1 | tail -15
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu 2>&1 | tail -2 > gpurun_out/bench_c2.txt
cat gpurun_out/bench_c2.txt
for w in c4 c3a c3b c1; do timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu 2>&1 | tail -1 > gpurun_out/bench_$w.txt; cut -c1-400 gpurun_out/bench_$w.txt; done
