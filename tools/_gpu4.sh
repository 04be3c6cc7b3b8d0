python bench.py --no-e2e --no-kmeans --no-cpu | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['kernel_ms'], d['clocks'])"
python bench.py --no-e2e --no-kmeans --no-cpu --steps 20 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['kernel_ms'], d['clocks'])"
