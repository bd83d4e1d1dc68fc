mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke4.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/gputests4.log 2>&1; echo tests=$?
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench4.json 2> gpurun_out/bench4.err; echo bench=$?
timeout 300 python bench.py --no-cpu-baseline --predictor mixed > gpurun_out/bench4m.json 2>&1; echo benchm=$?
