# split-K tail on/off per GEMM shape (tools/gemm_one.py names as arguments)
for n in "$@"; do
  python tools/gemm_one.py $n 6 | tail -1
  MT_GEMM_SPLITK=0 python tools/gemm_one.py $n 6 | tail -1 | sed 's/^/nosplit /'
done
