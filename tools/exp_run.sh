for c in 1 4 2; do
  python bench.py --config $c > gpurun_out/r1d_bench_cfg$c.json 2> gpurun_out/r1d_bench_cfg$c.err
done
