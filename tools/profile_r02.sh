#!/bin/bash
# Round-2 evidence for profiles/ (run under gpurun): bench line, launch lists of a c5 and a
# c4 step, and ncu --set full captures of the new library-free solver kernels and the small
# solver.  Usage: bash tools/profile_r02.sh
set -u
OUT=gpurun_out/r02
mkdir -p $OUT
python bench.py > $OUT/bench.json 2> $OUT/bench.err
CMD5="python tools/phase_timing.py --workload c5 --n-interior 3000 --reps 2"
CMD4="python tools/phase_timing.py --workload c4 --reps 3"
CMD1="python tools/phase_timing.py --workload c1 --reps 3"
$CMD5 > $OUT/phase_c5.json 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_c5_n3000.csv $CMD5 > $OUT/ncu_l5.log 2>&1
$CMD4 > $OUT/phase_c4.json 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_c4.csv $CMD4 > $OUT/ncu_l4.log 2>&1
$CMD1 > $OUT/phase_c1.json 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_c1.csv $CMD1 > $OUT/ncu_l1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_eig_large" -s 2 -c 1 -o $OUT/prof_eig_large $CMD5 > $OUT/ncu_a.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_dense_gemm" -s 20 -c 2 -o $OUT/prof_dense_gemm $CMD5 > $OUT/ncu_b.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_eig_mid" -s 4 -c 1 -o $OUT/prof_eig_mid $CMD4 > $OUT/ncu_c.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_gen_eig_small" -s 2 -c 1 -o $OUT/prof_eig_small $CMD1 > $OUT/ncu_d.log 2>&1
ls -la $OUT
