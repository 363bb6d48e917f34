mkdir -p gpurun_out
for n in g8_proj_fwd g4_proj_fwd g8_proj_dgrad g8_qkv_dgrad g8_fc1_dgrad g8_fc2_fwd qkv_fwd; do
  python tools/gemm_one.py $n 6 | tail -2
  MT_GEMM_SPLITK=0 python tools/gemm_one.py $n 6 | tail -1 | sed 's/^/nosplit /'
  MT_BN=128 python tools/gemm_one.py $n 6 | tail -1 | sed 's/^/bn128 /'
  MT_BN=192 python tools/gemm_one.py $n 6 | tail -1 | sed 's/^/bn192 /'
done
