mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke12.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -x -q -m gpu --durations=6 > gpurun_out/gputests12.log 2>&1; echo tests=$?
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench12.json 2> gpurun_out/bench12.err; echo bench=$?
timeout 600 python bench.py --no-cpu-baseline --config C3 --steps 3 > gpurun_out/bench12_c3.json 2>&1; echo c3=$?
timeout 600 python bench.py --no-cpu-baseline --config C5 --steps 3 > gpurun_out/bench12_c5.json 2>&1; echo c5=$?
