# cfg3: plan vs multi vs the flat kernel on one equally large tensor, four flush modes.
O=gpurun_out/r2b10; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python tools/probe_launch.py > $O/probe_launch.txt 2>&1; echo probe $?; cat $O/probe_launch.txt
