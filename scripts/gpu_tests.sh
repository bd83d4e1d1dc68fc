# GPU-box session: build, smoke, the -m gpu suite (fast part, then slow), one bench line.
# usage (from the repo root, under gpurun): bash scripts/gpu_tests.sh TAG ["pytest -k expr"]
TAG=${1:-t}
K=${2:-}
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo smoke=$?
if [ -n "$K" ]; then
  timeout 2400 python -m pytest tests -q -m gpu -k "$K" -s -rA > gpurun_out/${TAG}_tests.log 2>&1; echo tests=$?
else
  timeout 2400 python -m pytest tests -q -m "gpu and not slow" -s > gpurun_out/${TAG}_tests.log 2>&1; echo tests=$?
  timeout 2400 python -m pytest tests -q -m "gpu and slow" -s > gpurun_out/${TAG}_slow.log 2>&1; echo slow=$?
fi
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo bench=$?
tail -3 gpurun_out/${TAG}_tests.log
cat gpurun_out/${TAG}_bench.json | head -c 1500
