mkdir -p gpurun_out
timeout -k 10 900 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/gpu_gemm_pair.log 2>&1; echo rc=$? >> gpurun_out/gpu_gemm_pair.log
if grep -q "rc=0" gpurun_out/gpu_gemm_pair.log; then
for cl in 0 2; do BCMG_TCK_CLUSTER=$cl timeout 600 python tools/kernel_split.py --dtype f32 --n 65536 --t 1024 | sed "s/^{/{\"cluster\": $cl, /" >> gpurun_out/gemm_pair_split.jsonl; done
BCMG_TCK_CLUSTER=2 timeout 600 python tools/config_probe.py --config 5 --n 65536 --tiles 256,512,1024,2048 --dtypes f32,c64 --reps 2 > gpurun_out/config5_final.jsonl 2> gpurun_out/config5_final.err
fi
