# A/B of the wavefront host path: e2e of a workload for row-block heights and
# wavefront depths (DTB_WAVE_ROWS=0: plain H2D + passes + D2H)
wl=${1:-c3b}
run() {
  env $2 timeout 600 python bench.py --workload $1 --no-cpu --no-legs --steps 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1 $2 value', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
}
run $wl DTB_WAVE_ROWS=0
for v in "128 30" "96 40" "160 26" "128 44"; do set -- $v
  run $wl "DTB_WAVE_ROWS=$1 DTB_WAVE_PASSES=$2"
done
