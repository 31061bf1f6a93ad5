mkdir -p gpurun_out
: > gpurun_out/probe_pe.jsonl
for L in "" "$PWD/paper_2601_14466_b200/lib_probe1/libbcmg_b200.so"; do
  BCMG_LIB_PATH=$L timeout 600 python tools/kernel_split.py --dtype f32 --n 65536 --t 128 >> gpurun_out/probe_pe.jsonl 2>&1
  BCMG_LIB_PATH=$L timeout 600 python tools/kernel_split.py --dtype c64 --n 65536 --t 128 >> gpurun_out/probe_pe.jsonl 2>&1
done
