# A/B of the pipe kernel: current library vs ab/lib_base.so (the previous commit)
run() {
  env $2 timeout 600 python bench.py --workload $1 --no-cpu --no-legs --steps 3 --solve-steps ${3:-400} 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1 $2 value', round(d['value'],1), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
}
for i in 1 2; do for wl in c4 c3b; do
run $wl ""
run $wl DTB_LIB=ab/lib_base.so
done; done
DTB_LIB=ab/lib_probe.so python tools/pipe_probe.py 16384 16384 200 f64
