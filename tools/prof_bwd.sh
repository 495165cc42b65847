mkdir -p gpurun_out/bwdv
timeout 600 ncu --set full --import-source on --clock-control none -k regex:lstm_bwd_tc2v -c 1 -o gpurun_out/bwdv/v python tools/time_lstm_bwd_tc.py 128 > gpurun_out/bwdv/log 2>&1
DGC_BWD_EW=16 timeout 600 ncu --set full --import-source on --clock-control none -k regex:lstm_bwd_tc2w -c 1 -o gpurun_out/bwdv/w python tools/time_lstm_bwd_tc.py 128 >> gpurun_out/bwdv/log 2>&1
for k in v w; do ncu -i gpurun_out/bwdv/$k.ncu-rep --page raw --csv > gpurun_out/bwdv/${k}_raw.csv; ncu -i gpurun_out/bwdv/$k.ncu-rep --page source --csv > gpurun_out/bwdv/${k}_src.csv 2>/dev/null; done
ls -la gpurun_out/bwdv
