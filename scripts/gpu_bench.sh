# GPU-box session: the bench lines (ours N=1, the mlsort_sort_dist path at N=1, the reference
# arm), then ncu: the launch list of the bench command and one --set full capture each of the
# K1 and K3 kernels (after the same command exited 0 without ncu).  Reports are exported to
# CSV on the box and removed (gpurun_out/ must stay < 64 MiB).
# usage (repo root, under gpurun): bash scripts/gpu_bench.sh TAG [extra bench args]
TAG=${1:-b}
shift
EXTRA="$@"
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
timeout 900 python bench.py $EXTRA > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo bench=$?
if [ -z "$NODIST" ]; then
timeout 900 python bench.py --dist --config C4 --steps 3 --warmup 3 > gpurun_out/${TAG}_dist_c4.json 2> gpurun_out/${TAG}_dist_c4.err; echo dist=$?
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${TAG}_ref.json 2> gpurun_out/${TAG}_ref.err; echo ref=$?
fi
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline $EXTRA"
$CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu_launch.log 2>&1; echo ncu_launch=$?
for K in k1_ws k3_local; do
  S=3; KRE=k1_ws; [ $K = k3_local ] && S=6 && KRE="k3_local_sort<.*512"
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$KRE" -s $S -c 1 -o /tmp/${TAG}_$K $CMD > gpurun_out/${TAG}_ncu_$K.log 2>&1; echo ncu_$K=$?
  ncu -i /tmp/${TAG}_$K.ncu-rep --page raw --csv > gpurun_out/${TAG}_$K.raw.csv 2>&1
  ncu -i /tmp/${TAG}_$K.ncu-rep --page details --csv > gpurun_out/${TAG}_$K.details.csv 2>&1
  ncu -i /tmp/${TAG}_$K.ncu-rep --page source --csv > gpurun_out/${TAG}_$K.source.csv 2>&1
done
du -sh gpurun_out
head -c 3000 gpurun_out/${TAG}_bench.json; echo; head -c 1500 gpurun_out/${TAG}_dist_c4.json; echo; tail -3 gpurun_out/${TAG}_dist_c4.err
