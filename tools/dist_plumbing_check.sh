set -x
export KP_BENCH_DIST_BACKEND=gloo
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --scaling weak --steps 2 --warmup 3 --n-interior 2048 --n-boundary 600 --no-cpu > gpurun_out/dp2.log 2>&1; echo rc=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 4 --scaling weak --steps 2 --warmup 3 --n-interior 1024 --n-boundary 300 --no-cpu --optimizer kfac_star > gpurun_out/dp4s.log 2>&1; echo rc=$?
unset KP_BENCH_DIST_BACKEND
timeout 600 python bench.py --steps 2 --warmup 3 --n-interior 4096 --n-boundary 1200 --no-cpu > gpurun_out/dp1.log 2>&1; echo rc=$?
timeout 600 python bench.py --steps 2 --warmup 3 --n-interior 4096 --n-boundary 1200 --no-cpu --optimizer kfac_star > gpurun_out/dp1s.log 2>&1; echo rc=$?
for f in dp2 dp4s dp1 dp1s; do echo "== $f"; grep '^{' gpurun_out/$f.log | python -c "import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['n_gpus'], d['config']['n_interior_total'], d['config']['n_boundary_total'], d['losses_last_step'], d['e2e'] and d['e2e']['value'], d['value'])"; tail -3 gpurun_out/$f.log | cut -c1-300; done
