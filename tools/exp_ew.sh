timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for v in 16 12; do
  if [ $v = 16 ]; then export DGC_RNN_EW16=1; else unset DGC_RNN_EW16; fi
  echo "== EW $v"; python bench.py --steps 10 --warmup 3 --no-cpu-baseline --detail 2>&1 | grep -E "lstm|^\{" | cut -c1-160
done
