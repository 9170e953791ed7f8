mkdir -p gpurun_out
for c in c1 c2 c3 c5 c4; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/b_$c.json 2> gpurun_out/b_$c.err; echo "$c rc=$?"
done
