mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/gputest.log; cat gpurun_out/gputest.log
python profiles/ab_rebuild.py SWG_X=0 2>&1 | tee gpurun_out/ab5.log
for c in c5 c4; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b_$c.json 2> gpurun_out/b_$c.err; echo "$c rc=$?"
done
