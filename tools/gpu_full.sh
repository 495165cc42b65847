# full GPU suite + smoke + bench line
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -rf 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
cat gpurun_out/pytest_gpu.log gpurun_out/smoke.log; tail -c 300 gpurun_out/bench.json
