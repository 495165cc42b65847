# EvolveGCN weight-evolution kernel sweep on C3: parity per shape, then bench --detail.
for cl in ${@:-rr2 rr1 rr4 0}; do
  echo "== DGC_EVOLVE_CL=$cl"
  DGC_EVOLVE_CL=$cl timeout 600 python -m pytest tests/test_gpu_trainer.py -x -q -k evolve 2>&1 | tail -1
  DGC_EVOLVE_CL=$cl timeout 600 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline --detail > gpurun_out/evo_cl$cl.log 2>&1
  grep -E "^evolve" gpurun_out/evo_cl$cl.log; grep -o '"epoch_ms": [0-9.]*' gpurun_out/evo_cl$cl.log
done
