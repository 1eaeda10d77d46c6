cd /root/repo
TSG_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_2rank_gloo.log 2>&1; echo "rc=$?" >> gpurun_out/bench_2rank_gloo.log
TSG_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29556 bench.py --gpus 2 --steps 3 --warmup 3 --config rect --no-cpu-baseline > gpurun_out/bench_2rank_gloo_rect.log 2>&1; echo "rc=$?" >> gpurun_out/bench_2rank_gloo_rect.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "rc=$?" >> gpurun_out/bench_ref.log
