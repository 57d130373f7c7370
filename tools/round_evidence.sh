#!/bin/bash
# Round evidence on the GPU box: bench lines (all workloads + the reference
# arm), ncu launch lists of the bench commands, and one `ncu --set full`
# capture of each dominant kernel.  Output: gpurun_out/ev/ (summarised into
# profiles/ by tools/ncu_summary.py in the build container).
#   gpurun --timeout 3000 -- bash tools/round_evidence.sh [bench|launches|full|all]
set -u
what=${1:-all}
out=gpurun_out/ev
mkdir -p $out
NCU="ncu --clock-control none"
if [ "$what" = bench ] || [ "$what" = all ]; then
  timeout 900 python bench.py > $out/bench_c2.json 2> $out/bench_c2.err
  for w in c1 c3 c4; do
    timeout 900 python bench.py --workload $w > $out/bench_$w.json 2> $out/bench_$w.err
  done
  timeout 600 python bench.py --workload c2s --no-e2e --no-cpu --no-parity > $out/bench_c2s.json 2> $out/bench_c2s.err
  timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $out/bench_reference_c2.json 2> $out/bench_reference_c2.err
fi
if [ "$what" = launches ] || [ "$what" = all ]; then
  for w in c1 c2 c3 c4; do
    timeout 900 $NCU --metrics gpu__time_duration.sum -c 400 --csv --log-file $out/launches_$w.csv \
      python bench.py --workload $w --steps 3 --warmup 3 --no-e2e --no-cpu --no-parity --no-materialized > /dev/null 2>&1
  done
fi
if [ "$what" = full ] || [ "$what" = all ]; then
  timeout 900 $NCU --set full --import-source on -k regex:k_glm_fact_w -s 4 -c 1 -o $out/full_c2_fact \
    python bench.py --workload c2 --steps 3 --warmup 3 --no-e2e --no-cpu --no-parity --no-materialized > /dev/null 2>&1
  timeout 900 $NCU --set full --import-source on -k regex:k_glm_fact_w -s 6 -c 1 -o $out/full_c1_fact \
    python bench.py --workload c1 --steps 3 --warmup 3 --no-e2e --no-cpu --no-parity --no-materialized > /dev/null 2>&1
  timeout 900 $NCU --set full --import-source on -k regex:k_km_fact -s 4 -c 1 -o $out/full_c3_fact \
    python bench.py --workload c3 --steps 3 --warmup 3 --no-e2e --no-cpu --no-parity > /dev/null 2>&1
  timeout 900 $NCU --set full --import-source on -k regex:k_gnmf_t5 -s 4 -c 1 -o $out/full_c4_fact \
    python bench.py --workload c4 --steps 3 --warmup 3 --no-e2e --no-cpu --no-parity > /dev/null 2>&1
fi
# .ncu-rep files are too large to bring back (gpurun merges <= 64 MiB):
# summarise them here and keep the text
summarise() {
  for f in $out/full_*.ncu-rep; do
    [ -f "$f" ] || continue
    b=${f%.ncu-rep}
    python tools/ncu_summary.py report "$f" > "$b.txt" 2>&1
    python tools/ncu_source.py "$f" 40 >> "$b.txt" 2>&1
    rm -f "$f"
  done
}
summarise
ls -la $out
if [ "$what" = ops ]; then
  timeout 900 python tools/op_probe.py --crossprod c2 > $out/op_crossprod.txt 2>&1
  OP_KS=8,16,32 timeout 900 python tools/op_probe.py --wide c2 > $out/op_wide.txt 2>&1
  timeout 900 $NCU --metrics gpu__time_duration.sum --csv --log-file $out/launches_crossprod.csv \
    python tools/op_probe.py --crossprod c2 > /dev/null 2>&1
  OP_KS=32 timeout 900 $NCU --metrics gpu__time_duration.sum --csv --log-file $out/launches_wide32.csv \
    python tools/op_probe.py --wide c2 > /dev/null 2>&1
  timeout 900 $NCU --set full --import-source on -k regex:k_fgram_t5 -s 1 -c 1 -o $out/full_fgram \
    python tools/op_probe.py --crossprod c2 > /dev/null 2>&1
  OP_KS=32 timeout 900 $NCU --set full --import-source on -k regex:k_tmm_t5 -c 1 -o $out/full_tmm \
    python tools/op_probe.py --wide c2 > /dev/null 2>&1
  summarise
  ls -la $out
fi
