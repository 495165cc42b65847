make clean > /dev/null && make -j8 DGC_TS=1 > /dev/null 2>&1
timeout 200 python tools/time_lstm_c2.py 2>&1 | tail -2
timeout 200 python tools/time_lstm_fused.py 2>&1 | tail -9
make clean > /dev/null
