timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --detail 2>&1 | grep -E "a1b1|^\{" | cut -c1-130
