# Same-box A/B of compile-time macros under an environment: bash scripts/gpu_ab_env.sh "<flags A>" "<flags B>" "<ENV>" [bench args]
A="$1"; B="$2"; E="$3"; shift 3
for fl in "$A" "$B" "$A" "$B"; do
  MLSORT_NVCC_FLAGS="$fl" python -c "import paper_1805_04272_b200.build as b; b.build(force=True)" > /dev/null 2>&1
  env $E python bench.py --no-cpu-baseline "$@" 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('== [$fl] [$E]', round(d['ms_per_step'],4), 'ms  phases', [round(x,4) for x in r['phase_ms_mean']], 'frac', round(r['frac'],4))"
done
python -c "import paper_1805_04272_b200.build as b; b.build(force=True)" > /dev/null 2>&1
