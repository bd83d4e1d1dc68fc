# GPU-box session: one compute-sanitizer tool over the small product sorts of
# scripts/sanitize_sorts.py (n <= 2^16).  usage: bash scripts/gpu_sanitize.sh TAG TOOL [seconds]
# TOOL = racecheck | synccheck | memcheck (one tool per gpurun call: each replays every kernel).
TAG=${1:-san}; TOOL=${2:-racecheck}; T=${3:-900}
set -x
EXTRA=""
[ "$TOOL" = racecheck ] && EXTRA="--racecheck-report all"
MLSORT_NO_GRAPH=1 timeout $T compute-sanitizer --tool $TOOL $EXTRA --print-limit 50 python scripts/sanitize_sorts.py \
  > gpurun_out/${TAG}_${TOOL}.log 2>&1; echo ${TOOL}=$?
tail -40 gpurun_out/${TAG}_${TOOL}.log
