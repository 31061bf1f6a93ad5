mkdir -p gpurun_out
for n in 32768 65536; do timeout 600 python tools/kernel_split.py --dtype f64 --n $n --t 1024 >> gpurun_out/config2_split.jsonl 2>&1; done
timeout 600 python tools/kernel_split.py --dtype c128 --n 32768 --t 512 >> gpurun_out/config2_split.jsonl 2>&1
