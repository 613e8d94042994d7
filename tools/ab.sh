# A/B of experiment switches: bash tools/ab.sh "ENV1" "ENV2" ...  (one bench line each)
for e in "$@"; do
  echo "== $e"; env $e python bench.py --no-cpu --steps 10000 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1000,3),'us/step', round(d['value']/1e6,3),'M/s')"
done
