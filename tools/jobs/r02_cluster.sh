mkdir -p gpurun_out
timeout -k 5 600 python tools/cluster_check.py > gpurun_out/cluster_check.log 2>&1; echo rc=$? >> gpurun_out/cluster_check.log
if grep -q "rc=0" gpurun_out/cluster_check.log; then
  timeout -k 10 900 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/gpu_cluster.log 2>&1; echo rc=$? >> gpurun_out/gpu_cluster.log
  for cl in 0 2; do BCMG_TCK_CLUSTER=$cl timeout 600 python tools/config_probe.py --config 5 --n 65536 --tiles 512,1024,2048 --dtypes f32,c64 --reps 2 > gpurun_out/cluster_$cl.jsonl 2>gpurun_out/cluster_$cl.err; done
fi
