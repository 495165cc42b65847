# LSTM per-position timelines (timestamp build), then restore the production build
make clean > /dev/null && make -j8 DGC_TS=1 > /dev/null 2>&1
timeout 200 python tools/time_lstm_c2.py > gpurun_out/time_lstm_c2.txt 2>&1
timeout 200 python tools/time_lstm_fused.py > gpurun_out/time_lstm_fused.txt 2>&1
tail -4 gpurun_out/time_lstm_c2.txt; tail -3 gpurun_out/time_lstm_fused.txt
make clean > /dev/null
