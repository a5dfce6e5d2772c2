#!/bin/bash
# Build an A/B variant of libdtb_b200.so into ab/lib_<name>.so with extra
# -D defines (e.g. tools/build_variants.sh probe DTB_PIPE_PROBE=1). The
# timing-only exchange switches (DTB_NOPOLL, ...) live in
# tools/experiments/timing_only_exchange.patch.
set -e
cd "$(dirname "$0")/.."
mkdir -p ab
name=$1; shift
args=()
for d in "$@"; do args+=("-D$d"); done
python paper_2306_03336_b200/build.py "${args[@]}" --out=ab/lib_$name.so
