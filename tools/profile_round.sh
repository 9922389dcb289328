# One B200: the bench lines, the launch list and a full ncu capture of the
# dominant kernel (each ncu command only after the same command ran clean).
set -u
mkdir -p gpurun_out
python bench.py --steps 20 --warmup 5 > gpurun_out/p_bench_default.log 2>&1; echo "bench rc=$?" >> gpurun_out/p_summary.log
python bench.py --impl reference > gpurun_out/p_bench_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/p_summary.log
for c in 1 2 4; do python bench.py --config $c > gpurun_out/p_bench_c$c.log 2>&1; echo "c$c rc=$?" >> gpurun_out/p_summary.log; done
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-variants > gpurun_out/p_pre.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/p_launches.csv \
      python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-variants > gpurun_out/p_ncu1.log 2>&1
echo "launches rc=$?" >> gpurun_out/p_summary.log
python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-variants > gpurun_out/p_pre2.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:rollout_ozp -c 1 -o gpurun_out/p_ozp \
      python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-variants > gpurun_out/p_ncu2.log 2>&1
echo "full rc=$?" >> gpurun_out/p_summary.log
