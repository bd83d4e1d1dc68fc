mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
MLSORT_GROUP=1 timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/gputests10_group.log 2>&1; echo tests_group=$?
MLSORT_GROUP=1 timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench10_group.json 2> gpurun_out/bench10_group.err; echo bench_group=$?
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench10.json 2> gpurun_out/bench10.err; echo bench=$?
