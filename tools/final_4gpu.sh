#!/bin/bash
# Round-end multi-GPU evidence (gpurun --gpus 4): the full GPU suite once more, then bench lines at N=4 and N=2.
R=${R:-r02}
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --deselect tests/test_parity_bench.py > gpurun_out/${R}_gpu_tests_4gpu_final.log 2>&1; echo "suite rc=$?"; tail -2 gpurun_out/${R}_gpu_tests_4gpu_final.log
N=4 CFGS="gpt3 mtnlg pp 3d" STEPS=10 bash tools/multi_bench.sh
N=2 CFGS="gpt3 dp" STEPS=10 bash tools/multi_bench.sh
