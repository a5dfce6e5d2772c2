#!/bin/bash
# Build an A/B variant of libdtb_b200.so into ab/lib_<name>.so with extra
# -D defines (e.g. tools/build_variants.sh probe DTB_PIPE_PROBE=1). Timing-only
# switches (DTB_NOPOLL, DTB_NOREFRESH, DTB_NOPUBLISH, DTB_NOFENCE, DTB_NOSIDEPUB)
# build a library that solves only with DTB_TIMING_ONLY_OK=1 set.
set -e
cd "$(dirname "$0")/.."
mkdir -p ab
name=$1; shift
args=()
for d in "$@"; do args+=("-D$d"); done
python paper_2306_03336_b200/build.py "${args[@]}" --out=ab/lib_$name.so
