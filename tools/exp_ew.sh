python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --detail 2>&1 | cut -c1-130 | grep -E "gemm|softmax|reduce|^\{" 
