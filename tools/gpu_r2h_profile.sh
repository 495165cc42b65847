# round-2 final ncu evidence at C2 (launch list + --set full of the top kernels)
mkdir -p gpurun_out
bash tools/gpu_profile.sh r2h lstm_bwd_tc2k lstm_fwd_tc2v spmm_csr gemm_tf32_kernel > gpurun_out/prof_r2h.log 2>&1
head -30 gpurun_out/prof_r2h/launches_summary.txt
ls gpurun_out/prof_r2h
