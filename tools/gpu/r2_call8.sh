set -x
mkdir -p gpurun_out/r2
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 300 python tools/probe_zero.py; echo probe $?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:optim8bit_step -c 6 -o gpurun_out/r2/zero_vs_plain python tools/probe_zero.py --ncu > gpurun_out/r2/ncu_zero.log 2>&1; echo ncu $?
tail -3 gpurun_out/r2/ncu_zero.log
