mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke8.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/gputests8.log 2>&1; echo tests=$?
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench8.json 2> gpurun_out/bench8.err; echo bench=$?
MLSORT_FINE_BITS=13 timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench8_fb13.json 2> gpurun_out/bench8_fb13.err; echo bench13=$?
