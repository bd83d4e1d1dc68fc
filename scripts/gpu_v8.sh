# round-1 v8 evidence: bench line, ncu launch list, ncu section captures of K1 and K3
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/v8_smoke.log 2>&1; echo smoke=$?
timeout 600 python bench.py > gpurun_out/v8_bench.json 2> gpurun_out/v8_bench.err; echo bench=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/v8_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/v8_ncu.log 2>&1; echo ncu=$?
SKIP=1 bash scripts/gpu_prof.sh v8 k1_ws > /dev/null 2>&1; echo prof1=$?
SKIP=2 bash scripts/gpu_prof.sh v8 k3_local_sort > /dev/null 2>&1; echo prof3=$?
