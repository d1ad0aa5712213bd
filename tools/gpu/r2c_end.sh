# Final verification of HEAD: build + smoke, the whole GPU suite, the default bench line, the reference arm.
O=gpurun_out/r2c_end; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo smoke $?; tail -1 $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo pytest $?
tail -2 $O/pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo bench $?
python -c "import json; d=json.load(open('$O/bench.json')); print(d['ms_per_step'], d['roofline']['frac'], d['clocks'], d['e2e']['ms_per_step'])"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/ref.json 2> $O/ref.err; echo ref $?
