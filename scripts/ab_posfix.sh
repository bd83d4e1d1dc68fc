# A/B of K3's position-based fix-up (MLSORT_K3_POSFIX=0/1) on the C2 bench line, same box, then
# the -m gpu suite with the default build.  usage (under gpurun): bash scripts/ab_posfix.sh TAG
TAG=${1:-pf}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
for v in 0 1 0 1; do
  MLSORT_K3_POSFIX=$v MLSORT_DEBUG=1 timeout 600 python bench.py --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/${TAG}_$v.json 2> gpurun_out/${TAG}_$v.err
  python -c "
import json
d=json.loads(open('gpurun_out/${TAG}_$v.json').read()); r=d['roofline']
print('posfix=$v', round(d['ms_per_step'],4), 'ms', 'phases', [round(x,4) for x in r['phase_ms_mean']], d['info'])"
  grep -m1 "posfix_fallbacks" gpurun_out/${TAG}_$v.err
done
timeout 2400 python -m pytest tests -q -m "gpu and not slow" -x > gpurun_out/${TAG}_tests.log 2>&1; echo tests=$?
tail -3 gpurun_out/${TAG}_tests.log
