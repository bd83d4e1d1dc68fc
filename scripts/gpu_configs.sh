# GPU-box session: bench lines for the other BASELINE configs on one GPU (plan printed by
# MLSORT_DEBUG=1 on stderr).  usage: bash scripts/gpu_configs.sh TAG [configs...]
TAG=${1:-cfg}; shift
CFGS=${@:-C3 C5 C4}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
for c in $CFGS; do
  MLSORT_DEBUG=1 timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_$c.json 2> gpurun_out/${TAG}_$c.err
  echo "$c rc=$?"
  python -c "
import json
d=json.loads(open('gpurun_out/${TAG}_$c.json').read()); r=d['roofline']
print('$c', round(d['ms_per_step'],3), 'ms', 'phases', [round(x,3) for x in r['phase_ms_mean']], 'frac', round(r['frac'],4), d['info'])" 2>&1 | tail -1
  tail -2 gpurun_out/${TAG}_$c.err
done
