# A/B of resident-kernel build variants (DTB_LIB) on C2 / C3a
run() {
  env $2 timeout 600 python bench.py --workload $1 --no-cpu --no-legs --no-c5 --steps 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1 $2 value', round(d['value'],1), d['clocks']['sm_mhz'])"
}
for i in 1 2; do
run c2 ""; run c2 DTB_LIB=ab/lib_u16.so
run c3a ""; run c3a DTB_LIB=ab/lib_u8f32.so
done
