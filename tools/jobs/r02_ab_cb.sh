mkdir -p gpurun_out
: > gpurun_out/ab_cb.jsonl
for round in 1 2; do
for L in prev cur; do
  P=""; [ $L != cur ] && P=$PWD/paper_2601_14466_b200/lib_$L/libbcmg_b200.so
  BCMG_LIB_PATH=$P timeout 900 python tools/config_probe.py --config 5 --d 8 --tiles 512,1024 --reps 2 2>>gpurun_out/ab_cb.err | sed "s/^{/{\"lib\": \"$L\", /" >> gpurun_out/ab_cb.jsonl
done
done
