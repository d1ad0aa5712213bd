# cfg3 decomposition: ResNet-50 list vs block-rounded list vs one tensor through the plan vs the flat kernel.
O=gpurun_out/r2b14; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python tools/probe_multi.py > $O/probe_multi.txt 2>&1; echo probe $?; cat $O/probe_multi.txt
timeout 600 python tools/probe_multi.py > $O/probe_multi2.txt 2>&1; cat $O/probe_multi2.txt
