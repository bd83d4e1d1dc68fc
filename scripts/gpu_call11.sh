mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python bench.py --no-cpu-baseline --config C3 --steps 3 > gpurun_out/bench11_c3.json 2> gpurun_out/bench11_c3.err; echo c3=$?
MLSORT_GROUP=1 timeout 600 python bench.py --no-cpu-baseline --config C3 --steps 3 > gpurun_out/bench11_c3g.json 2> gpurun_out/bench11_c3g.err; echo c3g=$?
