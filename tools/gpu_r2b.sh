cd "$GRAFT_REPO_ROOT"
for l in "" build_variants/nohand.so build_variants/nocubes.so build_variants/nomacro.so; do
  VR_LIB=$l timeout 300 python tools/diag_c2.py 2>&1 | tail -9
done
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu2.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_gpu2.log
