mkdir -p gpurun_out
timeout -k 10 1200 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/gpu_subst.log 2>&1; echo rc=$? >> gpurun_out/gpu_subst.log
: > gpurun_out/potrs_phase2.jsonl
for V in 1 0; do
for a in "--dtype f32 --t 1024 --nrhs 1 --d 8" "--dtype f32 --t 128 --nrhs 1 --d 8" "--dtype c64 --t 1024 --nrhs 1 --d 8" "--dtype f64 --t 1024 --nrhs 4 --d 1" "--dtype c128 --t 512 --nrhs 4 --d 8"; do
  BCMG_SUBST_GEMV=$V timeout 300 python tools/potrs_phase.py --n 65536 $a | sed "s/^{/{\"gemv\": $V, /" >> gpurun_out/potrs_phase2.jsonl 2>>gpurun_out/potrs_phase2.err
done
done
timeout 900 python tools/config_probe.py --config 5 --d 8 --tiles 128,1024 --reps 2 > gpurun_out/c5_subst.jsonl 2> gpurun_out/c5_subst.err
