# A/B of end-to-end (render() from host) frame rate between library builds
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for r in 1 2; do for lib in build_variants/base.so build_variants/occ.so; do for c in c3 c1 c2; do
  VR_LIB=$lib timeout 300 python bench.py --config $c --steps 50 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', '$c', round(d['value'],1), 'e2e', round(d['e2e']['value'],1))"
done; done; done
