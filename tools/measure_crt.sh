#!/bin/bash
# Measurements of the INT8 tensor-core (CRT) line-search layer for profiles/ (run under gpurun):
# the tcgen05 int8 issue peak, the fold issue-rate probe, the layer micro-benchmark with its
# ablations and role timing for the three CTA organisations, one ncu --set full capture of the
# layer's kernels, and the launch list of whole bench steps.
# Usage: bash tools/measure_crt.sh r02   (binaries: see the build lines in tools/crt_bench.cu)
R=${1:-r02}
OUT=gpurun_out/$R/crt; mkdir -p $OUT
export LD_LIBRARY_PATH=$PWD/paper_2405_15603_b200
./tools/umma_i8_peak > $OUT/umma_i8_peak.txt 2>&1
./tools/fold_bench > $OUT/fold_bench.txt 2>&1
for c in 1 2 4; do
  echo "== KP_CRT_CLUSTER=$c, 768 -> 768, 16384 samples" >> $OUT/crt_bench.txt
  KP_CRT_CLUSTER=$c ./tools/crt_bench_timing 16384 768 768 100 3 >> $OUT/crt_bench.txt 2>&1
done
for shape in "768 512" "512 512"; do
  echo "== KP_CRT_CLUSTER=1, $shape, 16384 samples" >> $OUT/crt_bench.txt
  ./tools/crt_bench_timing 16384 $shape 100 3 >> $OUT/crt_bench.txt 2>&1
done
for v in nofold nomma none; do
  echo "== ablation $v (KP_CRT_CLUSTER=1, 768 -> 768)" >> $OUT/crt_bench.txt
  ./tools/crt_bench_$v 16384 768 768 100 2 >> $OUT/crt_bench.txt 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:k_crt -c 4 -o $OUT/crt_ncu \
  tools/crt_bench_full 16384 768 768 100 1 > $OUT/ncu_full.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file $OUT/launches_c5_n16384.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > $OUT/ncu_launches.log 2>&1
ls -la $OUT
