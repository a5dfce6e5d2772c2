#!/bin/bash
# A/B timing of library variants on C2 / C3a / C1 (resident) and C4 (pipe).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for lib in "$@"; do
  echo "== $lib"
  DTB_LIB=$lib python tools/sweep_bench.py 1900:1900:2000:f64:0:- 2700:2700:2000:f32:0:- 256:256:100:f64:0:- 2>&1 | cut -c1-220
done
