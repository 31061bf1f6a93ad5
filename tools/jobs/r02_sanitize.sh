# compute-sanitizer on small shapes, one tool per invocation (logs under gpurun_out/)
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for what in redist f64 f32 c64 loop; do
  timeout 900 $CS --tool memcheck --print-limit 20 python tools/sanitize_probe.py $what > gpurun_out/san_memcheck_$what.log 2>&1; echo rc=$? >> gpurun_out/san_memcheck_$what.log
done
for what in redist f64 f32; do
  timeout 1200 $CS --tool racecheck --racecheck-report analysis --print-limit 20 python tools/sanitize_probe.py $what > gpurun_out/san_racecheck_$what.log 2>&1; echo rc=$? >> gpurun_out/san_racecheck_$what.log
done
for what in redist f64; do
  timeout 900 $CS --tool synccheck --print-limit 20 python tools/sanitize_probe.py $what > gpurun_out/san_synccheck_$what.log 2>&1; echo rc=$? >> gpurun_out/san_synccheck_$what.log
done
