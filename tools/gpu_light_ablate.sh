# lighting on/off at c3 and c3soft (gradient + shading share of the frame), then the launch list
for c in c3 c3soft; do for l in true false; do
  timeout 300 python bench.py --config $c --steps 20 --no-cpu-baseline --no-e2e --set lighting=$l 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c lighting=$l', round(d['value'],1), 'fps', round(d['roofline']['kernel_ms'],3), 'ms', d['shaded_samples'], d['interpolated_samples'])"
done; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'visbits|vis_setup|aabb|box_kernel|count_hits|raycast' --csv --log-file gpurun_out/launches_setup.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo ncu=$?
