# A/B of the wavefront host path: e2e of C4 for row-block heights and
# wavefront depths (DTB_WAVE_ROWS=0: plain H2D + passes + D2H)
run() {
  env $2 timeout 600 python bench.py --workload $1 --no-cpu --no-legs --steps 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1 $2 value', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
}
for r in 128 192 256; do for m in 20 26 32; do
  run c4 "DTB_WAVE_ROWS=$r DTB_WAVE_PASSES=$m"
done; done
run c4 DTB_WAVE_ROWS=0
