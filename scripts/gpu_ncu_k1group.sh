# ncu --set full of the value-grouped K1 (MLSORT_GROUP=1) on the C2 bench step
TAG=${1:-kg}
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
MLSORT_GROUP=1 $CMD > gpurun_out/${TAG}_plain.json 2>&1 && \
MLSORT_GROUP=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k1_ws -s 3 -c 1 -o /tmp/${TAG} $CMD > gpurun_out/${TAG}_ncu.log 2>&1; echo ncu=$?
ncu -i /tmp/${TAG}.ncu-rep --page raw --csv > gpurun_out/${TAG}.raw.csv 2>&1
ncu -i /tmp/${TAG}.ncu-rep --page details --csv > gpurun_out/${TAG}.details.csv 2>&1
ncu -i /tmp/${TAG}.ncu-rep --page source --csv > gpurun_out/${TAG}.source.csv 2>&1
head -c 600 gpurun_out/${TAG}_plain.json
