# The full GPU suite on 4 GPUs, N times in a row (stability evidence), one log per run.
R=${R:-r02g}
for i in $(seq 1 ${N:-2}); do
  timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --deselect tests/test_parity_bench.py > gpurun_out/${R}_gpu_tests_4gpu_repeat$i.log 2>&1
  echo "run $i rc=$?"; tail -1 gpurun_out/${R}_gpu_tests_4gpu_repeat$i.log
done
