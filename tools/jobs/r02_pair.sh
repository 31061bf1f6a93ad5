# paired-panel tcgen05 trailing update: full GPU suite, then config 5 at T=128/256 with and without pairing
mkdir -p gpurun_out
timeout -k 10 900 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/gpu_pair.log 2>&1; echo rc=$? >> gpurun_out/gpu_pair.log
for pp in 0 1; do
  BCMG_PAIR_PANELS=$pp timeout 600 python tools/config_probe.py --config 5 --n 65536 --tiles 128,256,512 --dtypes f32,c64 --reps 2 > gpurun_out/pair_$pp.jsonl 2> gpurun_out/pair_$pp.err
done
