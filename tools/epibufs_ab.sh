# compile-time A/B: epilogue staging buffers per warp (2 = default) on the wgrad / forward GEMMs
for g in fc1_wgrad fc1_fwd qkv_fwd; do python tools/gemm_one.py $g 6 | tail -1; done
MT_NVCC_DEFINES="-DMT_GEMM_EPI_BUFS=4" python -m paper_2201_11990_b200.build > /dev/null
for g in fc1_wgrad fc1_fwd qkv_fwd; do echo -n "epi4 "; python tools/gemm_one.py $g 6 | tail -1; done
