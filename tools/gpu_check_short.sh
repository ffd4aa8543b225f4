# parity + default bench + a few configs on the current build
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), d['clocks'])"
CONFIGS="c3 c2 c1 c4" bash tools/variants.sh paper_2005_01442_b200/libvoxelray_b200.so
