#!/bin/bash
# Copy the latest capture_profiles.sh outputs (gpurun_out/) into profiles/r01/,
# regenerate the ncu summary and the bench tables of the docs.
set -e
cd "$(dirname "$0")/.."
cp gpurun_out/prof_resident.ncu-rep profiles/r01/resident_c2_2000steps.ncu-rep
cp gpurun_out/prof_pipe.ncu-rep profiles/r01/pipe_c4_1pass.ncu-rep
for w in c1 c2 c3a c3b c4 c5 ref; do cp gpurun_out/bench_$w.json profiles/r01/bench_$w.json; done
cp gpurun_out/launches_c2.csv profiles/r01/launches_bench_c2.csv
python tools/ncu_json.py profiles/r01/ncu_summary.json \
  "resident_kernel<double,4,8,0>=profiles/r01/resident_c2_2000steps.ncu-rep|python tools/sweep_bench.py 1900:1900:2000:f64:0:-  (ncu --set full --clock-control none -k regex:resident -c 1)|C2 geometry 1900x1900 fp64, 2000 steps, one launch" \
  "pipe_kernel<double,4,16,4,0>=profiles/r01/pipe_c4_1pass.ncu-rep|python tools/sweep_bench.py 16384:16384:8:f64:0:-  (ncu --set full --clock-control none -k regex:pipe -s 1 -c 1)|C4 geometry 16384x16384 fp64, one 8-step pass" > /dev/null
python tools/update_tables.py
