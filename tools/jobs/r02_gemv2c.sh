mkdir -p gpurun_out
AB_CASES=all timeout -k 5 900 python tools/ab_check.py BCMG_LIB_PATH "" $PWD/paper_2601_14466_b200/lib_ng/libbcmg_b200.so > gpurun_out/gemv2c_ab.log 2>&1; echo rc=$? >> gpurun_out/gemv2c_ab.log
: > gpurun_out/potrs_phase7.jsonl
for a in "--dtype c64 --t 1024 --nrhs 1 --d 8" "--dtype c64 --t 128 --nrhs 1 --d 8"; do
  timeout 300 python tools/potrs_phase.py --n 65536 $a >> gpurun_out/potrs_phase7.jsonl 2>>gpurun_out/potrs_phase7.err
done
