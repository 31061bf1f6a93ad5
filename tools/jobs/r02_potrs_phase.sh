mkdir -p gpurun_out
: > gpurun_out/potrs_phase.jsonl
timeout 300 python tools/potrs_phase.py --dtype f32 --n 65536 --t 1024 --nrhs 1 --d 8 >> gpurun_out/potrs_phase.jsonl 2>>gpurun_out/potrs_phase.err
timeout 300 python tools/potrs_phase.py --dtype f32 --n 65536 --t 128 --nrhs 1 --d 8 >> gpurun_out/potrs_phase.jsonl 2>>gpurun_out/potrs_phase.err
timeout 300 python tools/potrs_phase.py --dtype c64 --n 65536 --t 1024 --nrhs 1 --d 8 >> gpurun_out/potrs_phase.jsonl 2>>gpurun_out/potrs_phase.err
timeout 300 python tools/potrs_phase.py --dtype f64 --n 65536 --t 1024 --nrhs 64 --d 1 >> gpurun_out/potrs_phase.jsonl 2>>gpurun_out/potrs_phase.err
