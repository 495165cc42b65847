python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for v in 1 0; do
  if [ $v = 0 ]; then export DGC_GEMM_NO_TMA_STORE=1; fi
  echo "== tma_store $v"; python bench.py --steps 10 --warmup 3 --no-cpu-baseline --detail 2>&1 | grep -E "gemm|^\{" | cut -c1-150
done
