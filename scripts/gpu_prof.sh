# usage: bash scripts/gpu_prof.sh <tag> <kernel-regex> [<kernel-regex> ...]  -- ncu of the C2 bench step
mkdir -p gpurun_out
. scripts/ncu_sections.sh
tag=$1; shift
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline"
$B > gpurun_out/${tag}_plain.json 2>&1 || exit 1
for k in "$@"; do
  ncu $NCU_SECTIONS --clock-control none --import-source on -k regex:$k -s ${SKIP:-1} -c 1 -o /tmp/${tag}_$k $B > gpurun_out/${tag}_$k.log 2>&1
  ncu -i /tmp/${tag}_$k.ncu-rep --page details --csv > gpurun_out/${tag}_$k.details.csv 2>/dev/null
  ncu -i /tmp/${tag}_$k.ncu-rep --page source --csv --print-source sass > gpurun_out/${tag}_$k.source.csv 2>/dev/null
  ncu -i /tmp/${tag}_$k.ncu-rep --page raw --csv > gpurun_out/${tag}_$k.raw.csv 2>/dev/null
done
du -sh gpurun_out
