# What makes the weight-gradient GEMM slower than the forward: operand majors vs output type vs the
# short K (9216 tiles of K = 2048 instead of 1536 of K = 12288), and the tile width.
for g in fc1_fwd fwd_k2048 wg_kk_bf16 wg_km_bf16 wg_mk_bf16 wg_mm_bf16 wg_kk_f32 wg_mm_f32; do
  python tools/gemm_one.py $g 8 | tail -1
done
for bn in 128 192 256; do echo -n "BN=$bn "; MT_BN=$bn python tools/gemm_one.py wg_mm_f32 8 | tail -1; done
python tools/gemm_one.py wg_mm_f32 3 > /dev/null 2>&1 && \
  ncu --set full --import-source on --clock-control none -k regex:gemm_sm100 -s 2 -c 1 -o gpurun_out/r02_wgrad_dyn \
      python tools/gemm_one.py wg_mm_f32 3 > /dev/null 2>&1; echo "ncu rc=$?"
