python -m pytest tests -m gpu -x -q -k "lstm or tc" 2>&1 | tail -2
for pf in -1 0 1 2 4; do
  echo "PF=$pf"; DGC_RNN_PF=$pf python bench.py --steps 10 --warmup 3 --no-cpu-baseline --detail 2>&1 | grep -E "lstm|^\{" | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'): d=json.loads(l); print('  epoch ms', round(d['ms_per_step'],3))
    else: print('  ', l.strip())"
done
