# usage: tools/gpu_flag_ab.sh "<flags A>" "<flags B>" ... -> builds each variant lib, alternating probe + sustained bench
python -c "import __graft_entry__ as g; g.build()" > /dev/null
i=0; libs=()
for f in "$@"; do
  Q8_OBJDIR=/tmp/q8_f$i Q8_EXTRA_NVCC_FLAGS="$f" Q8_LIB_OUT=/tmp/libq8_f$i.so python paper_2110_02861_b200/build.py --force > /dev/null &
  libs+=(/tmp/libq8_f$i.so); i=$((i+1))
done
wait
for lib in "${libs[@]}"; do Q8_LIB_PATH=$lib timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "step_single or multi" 2>&1 | tail -1; done
bash tools/ab.sh "--iters 20" "${libs[@]}"
bash tools/ab_bench.sh "" "${libs[@]}"
