# A/B of library variants (visibility setup) + GPU parity tests + launch list of the setup kernels
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
CONFIGS="${CONFIGS:-c3 c2 c4}" bash tools/variants.sh ${VARIANTS:-build_variants/head.so build_variants/setup2.so build_variants/head.so build_variants/setup2.so}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'visbits|vis_setup|aabb|box_kernel|count_hits' --csv --log-file gpurun_out/launches_setup.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo ncu=$?
