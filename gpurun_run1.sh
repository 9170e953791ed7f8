mkdir -p gpurun_out/fin
for c in c1 c3 c4; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/fin/bench_$c.json 2> gpurun_out/fin/bench_$c.err; echo "$c rc=$?"
done
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/fin/ref_c5.json 2> gpurun_out/fin/ref_c5.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/fin/launches_c5.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/fin/ncu_c5.log 2>&1; echo "ncu rc=$?"
