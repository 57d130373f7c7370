out=gpurun_out/s3d; mkdir -p $out
for w in c1 c3; do
FL_BENCH_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 --workload $w --steps 5 --warmup 3 > $out/dist_$w.json 2> $out/dist_$w.err
echo "rc $?" >> $out/dist_$w.err
done
timeout 900 python bench.py --impl reference --workload c1 --steps 3 --warmup 1 > $out/ref_c1.json 2> $out/ref_c1.err
for w in c1 c3; do cut -c1-250 $out/dist_$w.json; tail -1 $out/dist_$w.err; done; cut -c1-250 $out/ref_c1.json
