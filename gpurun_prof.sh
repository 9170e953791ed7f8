mkdir -p gpurun_out
for c in c5; do
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,l1tex__t_sector_hit_rate.pct --clock-control none --csv --log-file gpurun_out/launch_$c.csv python bench.py --config $c --steps 1 --warmup 3 --no-graph --no-cpu-baseline --no-e2e > gpurun_out/ncu_$c.log 2>&1; echo "$c rc=$?"
done
