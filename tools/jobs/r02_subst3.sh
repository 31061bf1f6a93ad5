mkdir -p gpurun_out
: > gpurun_out/potrs_phase4.jsonl
for V in 1 0; do
for a in "--dtype f32 --t 1024 --nrhs 1 --d 8" "--dtype f32 --t 128 --nrhs 1 --d 8" "--dtype c64 --t 1024 --nrhs 1 --d 8" "--dtype f64 --t 1024 --nrhs 1 --d 1" "--dtype f64 --t 1024 --nrhs 4 --d 1" "--dtype c128 --t 512 --nrhs 1 --d 8" "--dtype c128 --t 512 --nrhs 4 --d 8" "--dtype f32 --t 256 --nrhs 2 --d 8"; do
  BCMG_SUBST_GEMV=$V timeout 300 python tools/potrs_phase.py --n 65536 $a | sed "s/^{/{\"gemv\": $V, /" >> gpurun_out/potrs_phase4.jsonl 2>>gpurun_out/potrs_phase4.err
done
done
