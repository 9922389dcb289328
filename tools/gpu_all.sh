mkdir -p gpurun_out
for f in tests/test_gpu_*.py; do
  b=$(basename $f .py)
  timeout 600 python -m pytest $f -q -x > gpurun_out/$b.log 2>&1
  echo "$b rc=$?" >> gpurun_out/summary.log
  tail -n1 gpurun_out/$b.log >> gpurun_out/summary.log
done
timeout 400 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/summary.log
timeout 300 python bench.py --config 1 > gpurun_out/bench_c1.log 2>&1; echo "c1 rc=$?" >> gpurun_out/summary.log
timeout 300 python bench.py --config 2 > gpurun_out/bench_c2.log 2>&1; echo "c2 rc=$?" >> gpurun_out/summary.log
