set -x
(nproc; free -g; lscpu | head -20; nvidia-smi) > gpurun_out/g1_box.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/g1_build.log 2>&1
timeout 1500 compute-sanitizer --tool racecheck --racecheck-report all python scripts/sanitize_sorts.py > gpurun_out/g1_racecheck.log 2>&1; echo racecheck=$?
tail -30 gpurun_out/g1_racecheck.log
