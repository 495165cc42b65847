# tests + smoke + bench (ours and the reference arm) on one B200
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
cat gpurun_out/pytest_gpu.log gpurun_out/smoke.log; tail -c 600 gpurun_out/bench.json; tail -c 400 gpurun_out/bench_reference.json
