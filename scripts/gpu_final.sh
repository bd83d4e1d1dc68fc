# GPU-box session for the measurement record: slow tests, the bench lines + ncu captures
# (gpu_bench.sh), the other configs (gpu_configs.sh).  usage: bash scripts/gpu_final.sh TAG
TAG=${1:-f}
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo smoke=$?
timeout 1200 python -m pytest tests -q -m "gpu and slow" > gpurun_out/${TAG}_slow.log 2>&1; echo slow=$?
tail -2 gpurun_out/${TAG}_slow.log
bash scripts/gpu_bench.sh ${TAG} 2>&1 | grep -E "^(bench|dist|ref|ncu)" 
bash scripts/gpu_configs.sh ${TAG}cfg C1 C3 C5 C4
