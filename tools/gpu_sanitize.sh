# compute-sanitizer memcheck / racecheck / synccheck over the hot kernels (small inputs)
mkdir -p gpurun_out/sanitize
for tool in memcheck racecheck synccheck; do
  for c in ${CASES:-sweep ecfimg stream cells_vb grid_hist grad}; do
    timeout 900 compute-sanitizer --tool $tool $( [ $tool = synccheck ] && echo "--num-cuda-barriers 64" ) --error-exitcode 9 --print-limit 20 python tools/sanitize_cases.py $c \
      > gpurun_out/sanitize/${tool}_${c}.log 2>&1
    echo "$tool $c rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|case .*: ok' gpurun_out/sanitize/${tool}_${c}.log | tr '\n' ' ')"
  done
done
