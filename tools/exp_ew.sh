timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | grep -E "^\{" | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), d['e2e'])"
