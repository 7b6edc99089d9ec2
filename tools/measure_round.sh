#!/bin/bash
# Round-end numbers for DESIGN.md / profiles (run under gpurun): the default bench line (with the
# CPU baseline and e2e), graph vs plain wall time per step and per-phase CUDA-event timings for
# c1-c4 at N = 3000, c5 at N = 3000 and 16384, KFAC* on c5.
# Usage: bash tools/measure_round.sh r02
R=${1:-r02}
OUT=gpurun_out/$R/final; mkdir -p $OUT
python bench.py > $OUT/bench_c5_n16384.json 2> $OUT/bench.err
python bench.py --optimizer kfac_star --no-cpu > $OUT/bench_c5_star_n16384.json 2>> $OUT/bench.err
for w in c1 c2 c3 c4; do python tools/step_timing.py --workload $w --steps 30 >> $OUT/step_timing.jsonl 2>&1; done
for w in c1 c2 c3 c4; do python tools/phase_timing.py --workload $w --reps 8 >> $OUT/phases.jsonl 2>&1; done
python tools/phase_timing.py --workload c5 --n-interior 3000 --reps 6 >> $OUT/phases.jsonl 2>&1
python tools/phase_timing.py --workload c5 --n-interior 16384 --reps 4 >> $OUT/phases.jsonl 2>&1
python tools/solve_timing.py --workload c5 --steps 2 --reps 2 > $OUT/solve_c5.jsonl 2>&1
python tools/solve_timing.py --workload c4 --steps 2 --reps 2 > $OUT/solve_c4.jsonl 2>&1
ls -la $OUT
python bench.py --n-interior 3000 --no-cpu > $OUT/bench_c5_n3000.json 2>> $OUT/bench.err
python bench.py --n-interior 65536 --no-cpu --steps 2 --warmup 3 > $OUT/bench_c5_n65536.json 2>> $OUT/bench.err
KP_CRT=0 python bench.py --no-cpu --no-e2e > $OUT/bench_c5_n16384_crt0.json 2>> $OUT/bench.err
