# Round-end bench lines only: tests, smoke, C2 (+ reference arm), C1, C3, C5 (when pushed)
bash tools/gpu_round.sh
bash tools/gpu_configs.sh > gpurun_out/configs.txt 2>&1
if [ -f artifacts/c5_graph.npz ]; then
  timeout 900 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline --detail > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
fi
