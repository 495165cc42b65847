python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-graph 2>&1 | grep -E "^\{" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('eager', d['ms_per_step'], d['e2e']['ms_per_step'])"
python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | grep -E "^\{" > gpurun_out/bench_graph.json; python -c "import json; d=json.load(open('gpurun_out/bench_graph.json')); print('graph', d['ms_per_step'], d['e2e']['ms_per_step'], d['gpu_launches'], d['roofline'])"
