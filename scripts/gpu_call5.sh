mkdir -p gpurun_out
. scripts/ncu_sections.sh
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline"
$B > gpurun_out/b5_plain.json 2>&1 && \
ncu $NCU_SECTIONS --clock-control none --import-source on -k regex:k1_ws -s 1 -c 1 -o /tmp/k1ws $B > gpurun_out/ncu_k1ws.log 2>&1; echo ncu1=$?
ncu $NCU_SECTIONS --clock-control none --import-source on -k regex:k3_local -s 1 -c 1 -o /tmp/k3v3 $B > gpurun_out/ncu_k3v3.log 2>&1; echo ncu3=$?
ls -la /tmp/*.ncu-rep
for r in k1ws k3v3; do
  ncu -i /tmp/$r.ncu-rep --page details --csv > gpurun_out/$r.details.csv 2>/dev/null
  ncu -i /tmp/$r.ncu-rep --page source --csv --print-source sass > gpurun_out/$r.source.csv 2>/dev/null
  ncu -i /tmp/$r.ncu-rep --page raw --csv > gpurun_out/$r.raw.csv 2>/dev/null
done
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o /tmp/k9 scripts/k9_pipes.cu && /tmp/k9 > gpurun_out/k9g.txt 2>&1; echo k9=$?
du -sh gpurun_out; ls -la gpurun_out | tail -12
