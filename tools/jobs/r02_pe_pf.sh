mkdir -p gpurun_out
: > gpurun_out/pe_pf.jsonl
for round in 1 2; do
for M in 0 1; do
  BCMG_EPI_MODE=$M timeout 600 python tools/kernel_split.py --dtype f32 --n 65536 --t 128 | sed "s/^{/{\"mode\": $M, /" >> gpurun_out/pe_pf.jsonl 2>&1
  BCMG_EPI_MODE=$M timeout 600 python tools/kernel_split.py --dtype c64 --n 65536 --t 128 | sed "s/^{/{\"mode\": $M, /" >> gpurun_out/pe_pf.jsonl 2>&1
done
done
