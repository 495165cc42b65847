# Round-end evidence: tests, smoke, all bench lines (C1/C2/C3; C5 when its artifacts were pushed),
# reference arm, C2 launch list, ncu --set full of the top kernels (C2 and C3)
bash tools/gpu_round.sh
bash tools/gpu_configs.sh > gpurun_out/configs.txt 2>&1
if [ -f artifacts/c5_graph.npz ]; then
  timeout 900 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline --detail > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
fi
bash tools/gpu_profile.sh final lstm_bwd_tc2k lstm_fwd_tc2v gemm_tf32 spmm_csr
bash tools/evo_profile.sh
bash tools/spmm_profile.sh
