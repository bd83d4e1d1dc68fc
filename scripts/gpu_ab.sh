# Same-box A/B of compile-time macros: usage bash scripts/gpu_ab.sh "<flags A>" "<flags B>" [bench args]
# Builds each variant in-tree, runs the C2 bench (no CPU baseline) twice per variant, prints
# ms/step and the phase times, then rebuilds the default.
A="$1"; B="$2"; shift 2
for fl in "$A" "$B" "$A" "$B"; do
  MLSORT_NVCC_FLAGS="$fl" python -c "import paper_1805_04272_b200.build as b; b.build(force=True)" > /dev/null 2>&1
  python bench.py --no-cpu-baseline --steps 20 "$@" 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('== [$fl]', round(d['ms_per_step'],4), 'ms  phases', [round(x,4) for x in r['phase_ms_mean']], 'frac', round(r['frac'],4))"
done
python -c "import paper_1805_04272_b200.build as b; b.build(force=True)" > /dev/null 2>&1
