# quick check: C2 bench line (k1/k3 ms), then the GPU tests
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('ms', d['ms_per_step'], 'k1', r['k1_ms'], 'k3', r['k3_ms'], 'phases', r['phase_ms_mean'], 'launches', d['gpu_launches'], d.get('info'))"
[ -n "$NOTEST" ] || timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
