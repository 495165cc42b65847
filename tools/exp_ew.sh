DGC_BWD_KSPLIT=1 timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python tools/time_lstm_bwd_tc.py 128 2>&1 | grep -E "ms|mean"
DGC_BWD_KSPLIT=1 timeout 300 python tools/time_lstm_bwd_tc.py 128 2>&1 | grep -E "ms|mean|rror"
DGC_BWD_KSPLIT=1 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --detail 2>&1 | grep -E "lstm|^\{" | cut -c1-200
