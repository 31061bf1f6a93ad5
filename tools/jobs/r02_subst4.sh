mkdir -p gpurun_out
: > gpurun_out/potrs_phase5.jsonl
for a in "--dtype f32 --t 1024 --nrhs 1 --d 8" "--dtype f32 --t 128 --nrhs 1 --d 8" "--dtype c64 --t 1024 --nrhs 1 --d 8" "--dtype c128 --t 512 --nrhs 1 --d 8" "--dtype f32 --t 256 --nrhs 2 --d 8"; do
  timeout 300 python tools/potrs_phase.py --n 65536 $a >> gpurun_out/potrs_phase5.jsonl 2>>gpurun_out/potrs_phase5.err
done
