#!/bin/bash
# One GPU call worth of evidence for profiles/: bench line, launch list (shares) and
# ncu --set full captures of the top kernels.  Usage (under gpurun):
#   bash tools/profile_round.sh r01
set -u
R=${1:-r01}
OUT=gpurun_out/$R
mkdir -p $OUT
python bench.py > $OUT/bench.json 2> $OUT/bench.err
CMD16="python tools/phase_timing.py --workload c5 --n-interior 16384 --reps 1"
$CMD16 > $OUT/phase16k.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_c5_n16384.csv $CMD16 > $OUT/ncu_launch.log 2>&1
# the bench workload's own launches (one line-search candidate: LOSS, LOSS, LAST) -> traffic per launch
ncu --set full --clock-control none -k regex:"k_gemm_act" -s 6 -c 3 -o $OUT/prof_gemm_act16k $CMD16 > $OUT/ncu0.log 2>&1
CMD3="python tools/phase_timing.py --workload c5 --n-interior 3000 --reps 1"
$CMD3 > $OUT/phase3k.log 2>&1 || exit 1
# launch order per step: accumulate (interior: 3 STORE; boundary: 3 STORE), line search k=0 (LOSS, LOSS, LAST ...)
ncu --set full --clock-control none --import-source on -k regex:"k_gemm_act" -s 6 -c 3 -o $OUT/prof_gemm_act $CMD3 > $OUT/ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_gemm_tn_tma" -s 1 -c 2 -o $OUT/prof_gemm_tn $CMD3 > $OUT/ncu2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_first_expand|k_act_bwd|k_gemm_nt_tma" -c 4 -o $OUT/prof_ew $CMD3 > $OUT/ncu3.log 2>&1
for w in c1 c2 c3 c4; do python tools/phase_timing.py --workload $w --n-interior 3000 --reps 5 >> $OUT/phases_small.jsonl 2>&1; done
ls -la $OUT
