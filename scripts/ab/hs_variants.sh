set -x
export PYTHONUNBUFFERED=1
python -c "import paper_2206_07896_b200" || exit 1
for v in 0 3 4 6 8; do
  BF_HOTSPOT_RING=$v timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k hotspot --timeout 200 2>&1 | tail -2
  BF_HOTSPOT_RING=$v timeout 300 python bench.py --steps 10 --warmup 3 --no-kernels --no-fused --no-cpu --no-bfs 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('RING', $v, d['value'], d['roofline']['frac'], d['ms_per_step'], d.get('clocks'))"
done
