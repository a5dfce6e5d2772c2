# A/B of resident-kernel build variants (DTB_LIB) on C2 / C3a / C1
run() {
  env $2 timeout 600 python bench.py --workload $1 --no-cpu --no-legs --no-c5 --steps 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1 $2 value', round(d['value'],1), d['clocks']['sm_mhz'])"
}
for i in 1 2 3; do
run c2 ""; run c2 DTB_LIB=ab/lib_fs1.so
run c3a ""; run c3a DTB_LIB=ab/lib_fs1.so
done
run c1 ""; run c1 DTB_LIB=ab/lib_fs1.so
