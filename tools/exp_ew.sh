timeout 600 python -m pytest tests -m gpu -x -q -k "spmm or trainer" 2>&1 | tail -2
for v in old new; do
  if [ $v = old ]; then export DGC_SPMM_OLD=1; else unset DGC_SPMM_OLD; fi
  echo "== $v"; python bench.py --steps 10 --warmup 3 --no-cpu-baseline --detail 2>&1 | grep -E "spmm|^\{" | cut -c1-160
done
