# Same-box A/B of prebuilt library variants (MLSORT_LIB): usage
#   bash scripts/ab_libs.sh "<variant> <variant> ..." [bench args]
# A variant is a library path ("default" = the in-tree libmlsort.so), optionally followed by
# ":VAR=value[,VAR=value]" environment settings.  Runs the bench (no CPU baseline) twice per
# variant, interleaved, and prints ms/step, the phase times and the K1 roofline fraction.
VARIANTS="$1"; shift
for rep in 1 2; do
  for V in $VARIANTS; do
    L="${V%%:*}"; E=""
    [ "$V" != "$L" ] && E="${V#*:}" && E="${E//,/ }"
    [ "$L" != default ] && E="MLSORT_LIB=$L $E"
    env $E python bench.py --no-cpu-baseline --steps 20 "$@" 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('== [$V $*]', round(d['ms_per_step'],4), 'ms  phases', [round(x,4) for x in r['phase_ms_mean']], 'frac', round(r['frac'],4), flush=True)"
  done
done
