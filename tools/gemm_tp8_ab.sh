# TP=8 projection GEMMs: tile widths and all-tile split-K (MT_GEMM_SPLIT_ALL) vs the default
python tools/gemm_tp8_shapes.py 2>&1 | grep -v cuBLAS
for sa in 2 3 4; do echo "MT_GEMM_SPLIT_ALL=$sa"; MT_GEMM_SPLIT_MINK=64 MT_GEMM_SPLIT_ALL=$sa python tools/gemm_tp8_shapes.py 2>&1 | grep -v cuBLAS | grep "bn=0"; done
