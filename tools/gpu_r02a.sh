mkdir -p gpurun_out/r02a
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02a/smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02a/pytest_gpu.txt 2>&1
echo "pytest exit $?" >> gpurun_out/r02a/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02a/smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/r02a/bench_c2.json 2> gpurun_out/r02a/bench_c2.err
timeout 900 python bench.py --impl reference > gpurun_out/r02a/bench_ref.json 2> gpurun_out/r02a/bench_ref.err
