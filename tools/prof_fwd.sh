mkdir -p gpurun_out/fwdx
timeout 600 ncu --set full --import-source on --clock-control none -k regex:lstm_fwd_tc2v -c 1 -o gpurun_out/fwdx/f python tools/time_lstm_fused.py > gpurun_out/fwdx/log 2>&1
ncu -i gpurun_out/fwdx/f.ncu-rep --page raw --csv > gpurun_out/fwdx/f_raw.csv
ncu -i gpurun_out/fwdx/f.ncu-rep --page source --csv > gpurun_out/fwdx/f_src.csv 2>/dev/null
ls -la gpurun_out/fwdx
