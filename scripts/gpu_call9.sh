mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke9.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/gputests9.log 2>&1; echo tests=$?
timeout 300 python bench.py > gpurun_out/bench9.json 2> gpurun_out/bench9.err; echo bench=$?
python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/b9_plain.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches9.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu9.log 2>&1; echo ncu=$?
