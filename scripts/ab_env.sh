# A/B of env-switched variants on one bench config, same box, interleaved twice.
# usage (under gpurun): bash scripts/ab_env.sh TAG CONFIG "ENV_A" "ENV_B" ...   ("-" = no env)
TAG=$1; CFG=$2; shift 2
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
for rep in 1 2; do
i=0
for E in "$@"; do
  i=$((i+1)); EE="$E"; [ "$E" = "-" ] && EE=""
  env $EE timeout 600 python bench.py --config $CFG --no-cpu-baseline --steps 40 --warmup 5 > gpurun_out/${TAG}_$i.json 2> gpurun_out/${TAG}_$i.err
  python -c "
import json
d=json.loads(open('gpurun_out/${TAG}_$i.json').read()); r=d['roofline']
print('$CFG [$E]', round(d['ms_per_step'],4), 'ms', 'phases', [round(x,4) for x in r['phase_ms_mean']], d['info'].get('repairs'))"
done
done
