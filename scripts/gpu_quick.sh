# GPU-box session: C2 bench line (40 steps), then the -m gpu suite (fast part, stop at the first
# failure).  usage (under gpurun): bash scripts/gpu_quick.sh TAG
TAG=${1:-q}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
for i in 1 2; do
timeout 600 python bench.py --no-cpu-baseline --steps 40 --warmup 5 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo bench=$?
python -c "
import json
d=json.loads(open('gpurun_out/${TAG}_bench.json').read()); r=d['roofline']
print('C2', round(d['ms_per_step'],4), 'ms', 'phases', [round(x,4) for x in r['phase_ms_mean']], d['info'])"
done
timeout 2400 python -m pytest tests -q -m "gpu and not slow" -x > gpurun_out/${TAG}_tests.log 2>&1; echo tests=$?
tail -5 gpurun_out/${TAG}_tests.log
