# A/B of the pipe kernel: current library vs ab/lib_base2.so (the previous commit)
run() {
  env $2 timeout 900 python bench.py --workload $1 --no-cpu --no-legs --no-strong --steps 3 ${3:+--solve-steps $3} 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1 $2 value', round(d['value'],1), 'e2e', round((d.get('e2e') or {}).get('value',0),1), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
}
for i in 1 2; do
run c4 "" ; run c4 DTB_LIB=ab/lib_base2.so
run c5 "" ; run c5 DTB_LIB=ab/lib_base2.so
done
for i in 1 2; do run c3b ""; run c3b DTB_LIB=ab/lib_base2.so; done
DTB_LIB=ab/lib_probe.so python tools/pipe_probe.py 16384 16384 200 f64; DTB_LIB=ab/lib_probe.so python tools/pipe_probe.py 8192 8192 200 f32
