out=gpurun_out/r02t; mkdir -p $out
for dg in 0 1 2 3; do
  FL_GN5_DIAG=$dg timeout 600 python bench.py --workload c4 --steps 10 --no-e2e --no-cpu --no-parity > $out/bench_c4_diag$dg.json 2> $out/bench_c4_diag$dg.err
done
