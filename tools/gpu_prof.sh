#!/bin/bash
# Trace + ncu captures of the resident (C2) and pipe (C4) kernels.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
DTB_TRACE=1 python tools/sweep_bench.py 1900:1900:2000:f64:0:- 1900:1900:10000:f64:0:- 2700:2700:2000:f32:0:- > gpurun_out/trace_res.log 2>&1
cat gpurun_out/trace_res.log
ncu --set full --import-source on --clock-control none -k regex:resident -c 1 \
    -o gpurun_out/prof_resident python tools/sweep_bench.py 1900:1900:2000:f64:0:- \
    > gpurun_out/ncu_res.log 2>&1
echo "ncu resident rc=$?"
ncu --set full --import-source on --clock-control none -k regex:pipe -s 1 -c 1 \
    -o gpurun_out/prof_pipe python tools/sweep_bench.py 16384:16384:8:f64:0:- \
    > gpurun_out/ncu_pipe.log 2>&1
echo "ncu pipe rc=$?"
