#!/bin/bash
# Round evidence on one B200: bench lines for every workload, the ncu launch
# list of the headline bench command, and full ncu captures of the resident
# (C2, C3a) and pipelined (C4) kernels. Outputs land in gpurun_out/ and are
# summarised into profiles/<round>/ by hand (tools/ncu_json.py, ncu_summary.py).
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
echo "c2 rc=$?"
for w in c1 c3a c3b c4 c5; do
  python bench.py --workload $w --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
  echo "$w rc=$?"
done
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
echo "ref rc=$?"
# launch list of the headline command (kernel share, cold-cache serialised times)
python bench.py --steps 2 --warmup 3 --no-cpu --no-legs --no-c5 > gpurun_out/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-legs --no-c5 \
    > gpurun_out/ncu_launches.log 2>&1
echo "launches rc=$?"
# full captures of the main kernels (each command first run plain, exit 0)
python tools/sweep_bench.py 1900:1900:2000:f64:0:- > gpurun_out/plain_res.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:resident -c 1 \
    -o gpurun_out/prof_resident_c2 python tools/sweep_bench.py 1900:1900:2000:f64:0:- \
    > gpurun_out/ncu_res.log 2>&1
echo "ncu resident c2 rc=$?"
python tools/sweep_bench.py 2700:2700:2000:f32:0:- > gpurun_out/plain_res32.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:resident -c 1 \
    -o gpurun_out/prof_resident_c3a python tools/sweep_bench.py 2700:2700:2000:f32:0:- \
    > gpurun_out/ncu_res32.log 2>&1
echo "ncu resident c3a rc=$?"
python tools/sweep_bench.py 16384:16384:8:f64:0:- > gpurun_out/plain_pipe.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:pipe -s 1 -c 1 \
    -o gpurun_out/prof_pipe_c4 python tools/sweep_bench.py 16384:16384:8:f64:0:- \
    > gpurun_out/ncu_pipe.log 2>&1
echo "ncu pipe rc=$?"
# phase traces
DTB_TRACE=1 python tools/sweep_bench.py 1900:1900:10000:f64:0:- 2700:2700:10000:f32:0:- \
    256:256:100:f64:0:- > gpurun_out/trace_res.log 2>&1
echo "trace rc=$?"
