python -m pytest tests -m gpu -x -q -k "lstm or tc or trainer" 2>&1 | tail -2
for ew in 16 v; do
  echo "== FWD $ew"; if [ $ew = v ]; then unset DGC_FWD_EW; else export DGC_FWD_EW=$ew; fi; python tools/time_lstm_tc.py 128 2>&1 | grep -E "^tc|per-step"
done
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --detail 2>&1 | grep -E "lstm|^\{" | cut -c1-200
