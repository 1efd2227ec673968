timeout 300 python -m pytest tests -m gpu -q --timeout 120 -x > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
for k in flat split; do
echo -n "$k " >> gpurun_out/variants10.log
NVC_QUERY_KERNEL=$k timeout 120 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['ms_per_step'], d['config']['stage_ms'])" >> gpurun_out/variants10.log 2>&1
done
