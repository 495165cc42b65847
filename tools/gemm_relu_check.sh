# C2/C3 detail tables (relu-masked GEMM epilogue prefetch A/B)
for c in c3 c2; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --detail > gpurun_out/gr_$c.json 2>gpurun_out/gr_$c.err; grep -E "gemm" gpurun_out/gr_$c.err | head -8; grep -o '"epoch_ms": [0-9.]*' gpurun_out/gr_$c.json; done
