mkdir -p gpurun_out
: > gpurun_out/epi_mode_check.log
for M in 1 2 3; do BCMG_TCK_EPI=1 timeout -k 5 600 python tools/ab_check.py BCMG_EPI_MODE 0 $M >> gpurun_out/epi_mode_check.log 2>&1; echo rc=$? >> gpurun_out/epi_mode_check.log; done
for M in 0 1 2 3; do
  BCMG_EPI_MODE=$M timeout 600 python tools/kernel_split.py --dtype f32 --n 65536 --t 128 > gpurun_out/mode_f32_$M.jsonl 2>&1
  BCMG_EPI_MODE=$M BCMG_TCK_EPI=1 timeout 600 python tools/kernel_split.py --dtype c64 --n 65536 --t 128 > gpurun_out/mode_c64_$M.jsonl 2>&1
done
