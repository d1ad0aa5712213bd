python -c "import __graft_entry__ as g; g.build()" > /dev/null
Q8_OBJDIR=/tmp/q8_alt Q8_EXTRA_NVCC_FLAGS="-DQ8_QT_MIN_K=$1" Q8_LIB_OUT=/tmp/libq8_alt.so python paper_2110_02861_b200/build.py --force > /dev/null
timeout 600 python -m pytest tests/test_gpu_quantiles.py -x -q 2>&1 | tail -2
Q8_LIB_PATH=/tmp/libq8_alt.so timeout 600 python -m pytest tests/test_gpu_quantiles.py -x -q 2>&1 | tail -2
for rep in 1 2; do
for lib in paper_2110_02861_b200/libq8.so /tmp/libq8_alt.so; do
Q8_LIB_PATH=$lib python bench.py --workload quantiles_gpt2_xl --steps 20 --warmup 3 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', round(d['ms_per_step'],3), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])"
done; done
