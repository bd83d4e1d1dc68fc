# A/B of K3's position-based fix-up with and without the CUDA-graph path, 40 timed steps each,
# then the ncu launch list of both.  usage (under gpurun): bash scripts/ab_posfix2.sh TAG
TAG=${1:-pf}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
for g in graph nograph; do
for v in 0 1 0 1; do
  E=""; [ $g = nograph ] && E="MLSORT_NO_GRAPH=1"
  env $E MLSORT_K3_POSFIX=$v timeout 600 python bench.py --no-cpu-baseline --steps 40 --warmup 5 > gpurun_out/${TAG}_${g}_$v.json 2> gpurun_out/${TAG}_${g}_$v.err
  python -c "
import json
d=json.loads(open('gpurun_out/${TAG}_${g}_$v.json').read()); r=d['roofline']
print('$g posfix=$v', round(d['ms_per_step'],4), 'ms', 'phases', [round(x,4) for x in r['phase_ms_mean']])"
done
done
for v in 0 1; do
MLSORT_K3_POSFIX=$v timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/${TAG}_launches_$v.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_ncu_$v.log 2>&1
python scripts/launch_summary.py gpurun_out/${TAG}_launches_$v.csv 2>&1 | head -8
done
