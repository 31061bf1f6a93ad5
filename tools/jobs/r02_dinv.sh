mkdir -p gpurun_out
: > gpurun_out/dinv3.log
for cfg in "N=640 T=64" "N=649 T=64" "N=1100 T=96" "N=2048 T=128" "N=700 T=128"; do
  echo "== $cfg" >> gpurun_out/dinv3.log
  env $cfg timeout 300 python tools/dinv_debug.py >> gpurun_out/dinv3.log 2>&1
done
