timeout 2400 python -m pytest tests -m gpu -q -x --timeout 1500 2>&1 | tail -6
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
