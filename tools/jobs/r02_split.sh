mkdir -p gpurun_out
for spec in "f32 65536 1024" "f32 65536 128" "c64 65536 1024" "f32 65536 512"; do set -- $spec
  timeout 600 python tools/kernel_split.py --dtype $1 --n $2 --t $3 >> gpurun_out/kernel_split.jsonl 2>> gpurun_out/kernel_split.err
done
