cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --dist-backend gloo --steps 2 --warmup 3 --no-cpu > gpurun_out/bench_gloo2.json 2> gpurun_out/bench_gloo2.err; echo "rc=$?" >> gpurun_out/bench_gloo2.err
timeout 900 python bench.py --force-dist --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_fd.json 2> gpurun_out/bench_fd.err; echo "rc=$?" >> gpurun_out/bench_fd.err
tail -5 gpurun_out/bench_gloo2.err; cut -c1-1500 gpurun_out/bench_gloo2.json; tail -2 gpurun_out/bench_fd.err; cut -c1-600 gpurun_out/bench_fd.json
