mkdir -p gpurun_out
timeout -k 5 900 python tools/ab_check.py BCMG_TCK_PAIR_EPI 1 3 > gpurun_out/quarter_ab.log 2>&1; echo rc=$? >> gpurun_out/quarter_ab.log
if grep -q "rc=0" gpurun_out/quarter_ab.log; then
: > gpurun_out/quarter.jsonl
for U in 1 3; do
  BCMG_TCK_PAIR_EPI=$U timeout 600 python tools/kernel_split.py --dtype f32 --n 65536 --t 128 | sed "s/^{/{\"pe\": $U, /" >> gpurun_out/quarter.jsonl 2>&1
  BCMG_TCK_PAIR_EPI=$U timeout 600 python tools/kernel_split.py --dtype c64 --n 65536 --t 128 | sed "s/^{/{\"pe\": $U, /" >> gpurun_out/quarter.jsonl 2>&1
done
fi
