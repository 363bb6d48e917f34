# A/B: relaxed vs release remote arrive in the GEMM epilogue (launch list of one bench step each)
python bench.py --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -s 40 -c 40 --csv --log-file gpurun_out/ab_relaxed.csv python bench.py --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
MT_NVCC_DEFINES="-DMT_GEMM_RELEASE_ARRIVE=1" python -m paper_2201_11990_b200.build > /dev/null
ncu --metrics gpu__time_duration.sum --clock-control none -s 40 -c 40 --csv --log-file gpurun_out/ab_release.csv python bench.py --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
python -m paper_2201_11990_b200.build > /dev/null   # back to the default build for the bench lines
for r in 1 2; do
  python bench.py --steps 20 --warmup 5 --no-cpu | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('relaxed', round(d['ms_per_step'],3), d['clocks']['sm_mhz'])"
  MT_NVCC_DEFINES="-DMT_GEMM_RELEASE_ARRIVE=1" python -m paper_2201_11990_b200.build > /dev/null
  python bench.py --steps 20 --warmup 5 --no-cpu | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('release', round(d['ms_per_step'],3), d['clocks']['sm_mhz'])"
  python -m paper_2201_11990_b200.build > /dev/null
done
