# A/B of block red-black kernel builds on one box (development aid): bash tools/ab_bp.sh libA libB ...
for lib in "$@"; do
  for B in 1 2 4 8 16; do
    SOR_LIBRARY=$lib timeout 200 python bench.py --method block --block $B --steps 3 --warmup 1 2>/dev/null \
      | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$lib B=$B', round(d['value'],1), 'GLUP/s frac', round(d['roofline']['frac'],3))"
  done
done
