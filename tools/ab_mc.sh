# A/B of multi-colour kernel builds on one box (development aid): bash tools/ab_mc.sh libA libB ...
for lib in "$@"; do
  for col in 1,1,4 1,1,2 1,2,3 5,2,8; do
    SOR_LIBRARY=$lib timeout 200 python bench.py --method multicolor --colours $col --steps 3 --warmup 1 2>/dev/null \
      | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$lib $col', round(d['value'],1), 'GLUP/s frac', round(d['roofline']['frac'],3))"
  done
done
