# round 2: launch list + ncu --set full of the top kernels at C2; LSTM timelines
mkdir -p gpurun_out
bash tools/gpu_profile.sh r2b lstm_bwd_tc2k lstm_fwd_tc2v spmm_csr > gpurun_out/prof_r2b.log 2>&1
cat gpurun_out/prof_r2b/launches_summary.txt | head -20
make clean > /dev/null && make -j8 DGC_TS=1 > /dev/null 2>&1
timeout 300 python tools/time_lstm_c2.py > gpurun_out/time_lstm_c2.txt 2>&1
timeout 300 python tools/time_lstm_fused.py > gpurun_out/time_lstm_fused.txt 2>&1
tail -3 gpurun_out/time_lstm_c2.txt; tail -3 gpurun_out/time_lstm_fused.txt
make clean > /dev/null
