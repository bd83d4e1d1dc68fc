# GPU-box session: one config under several environment variants (plan / variant switches).
# usage: bash scripts/gpu_envs.sh TAG CONFIG "ENV1" "ENV2" ...   (ENV "" = default)
TAG=$1; CFG=$2; shift 2
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
for e in "$@"; do
  env $e MLSORT_DEBUG=1 timeout 600 python bench.py --config $CFG --steps 3 --warmup 2 --no-cpu-baseline > /tmp/o.json 2> /tmp/o.err
  python -c "
import json
d=json.loads(open('/tmp/o.json').read()); r=d['roofline']
print('[$e]', '$CFG', round(d['ms_per_step'],3), 'ms phases', [round(x,3) for x in r['phase_ms_mean']], d['info'])" 2>&1 | tail -1
  grep "plan" /tmp/o.err | tail -1
done
