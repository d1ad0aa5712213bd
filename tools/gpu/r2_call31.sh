python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 300 python tools/probe_launch.py
