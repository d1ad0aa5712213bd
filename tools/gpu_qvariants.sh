# usage: tools/gpu_qvariants.sh "<flags A>" "<flags B>" ...  -> builds each variant, runs the quantile tests on the
# first, benches all twice (SRAM-Quantiles workload)
python -c "import __graft_entry__ as g; g.build()" > /dev/null
i=0; libs=()
for f in "$@"; do
  Q8_OBJDIR=/tmp/q8_v$i Q8_EXTRA_NVCC_FLAGS="$f" Q8_LIB_OUT=/tmp/libq8_v$i.so python paper_2110_02861_b200/build.py --force > /dev/null &
  libs+=(/tmp/libq8_v$i.so); i=$((i+1))
done
wait
for lib in "${libs[@]}"; do Q8_LIB_PATH=$lib timeout 600 python -m pytest tests/test_gpu_quantiles.py -x -q 2>&1 | tail -1; done
for rep in 1 2; do i=0
for lib in "${libs[@]}"; do
Q8_LIB_PATH=$lib python bench.py --workload quantiles_gpt2_xl --steps 20 --warmup 3 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('v$i', round(d['ms_per_step'],3), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])"; i=$((i+1))
done; done
