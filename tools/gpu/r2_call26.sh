python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
echo default; timeout 300 python tools/probe_launch.py 2>&1 | grep multi
echo ns3x256; Q8_NSUB=3 Q8_SUBT=256 timeout 300 python tools/probe_launch.py 2>&1 | grep multi
echo ns2x256; Q8_NSUB=2 Q8_SUBT=256 timeout 300 python tools/probe_launch.py 2>&1 | grep multi
echo ns3x128; Q8_NSUB=3 Q8_SUBT=128 timeout 300 python tools/probe_launch.py 2>&1 | grep multi
