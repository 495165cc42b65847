timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --detail 2>&1 | grep -E "lstm|gemm|spmm|^\{" | cut -c1-130
