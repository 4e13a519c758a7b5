# C3 at T=5: solve-phase check mode 3 (all cells, high words) vs 4 (probe rows)
for ck in 3 4; do
SOR_SOLVE_CK=$ck python bench.py --T 5 --no-c5 --no-small --steps 5 --warmup 3 2>/dev/null > /tmp/b.json
python - $ck <<'PY'
import json, sys
l = json.loads(open('/tmp/b.json').read().strip().splitlines()[-1])
print("ck", sys.argv[1], "T", l["config"]["temporal_depth"], round(l["value"], 1), round(l["fixed_phase_glups"], 1),
      round(l["solve_phase_glups"], 1), l["clocks"]["sm_mhz"])
PY
done
