mkdir -p gpurun_out
timeout -k 5 900 python tools/ab_check.py BCMG_LIB_PATH "" $PWD/paper_2601_14466_b200/lib_ng/libbcmg_b200.so > gpurun_out/gemv4_ab.log 2>&1; echo rc=$? >> gpurun_out/gemv4_ab.log
: > gpurun_out/potrs_phase6.jsonl
for a in "--dtype f32 --t 1024 --nrhs 1 --d 8" "--dtype f32 --t 128 --nrhs 1 --d 8"; do
  timeout 300 python tools/potrs_phase.py --n 65536 $a >> gpurun_out/potrs_phase6.jsonl 2>>gpurun_out/potrs_phase6.err
done
