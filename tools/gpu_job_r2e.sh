set -x
mkdir -p gpurun_out
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 \
  bench.py --gpus 2 --dist-backend gloo --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_w2_gloo.json 2> gpurun_out/bench_w2_gloo.err
echo w2 rc=$?; tail -c 800 gpurun_out/bench_w2_gloo.json
timeout 1200 python bench.py --config 4 --steps 1 --warmup 1 --no-cpu --no-e2e --no-fp64 --layout-iters 20 > gpurun_out/bench_c4_1gpu.json 2> gpurun_out/bench_c4_1gpu.err
echo c4 rc=$?; tail -c 1200 gpurun_out/bench_c4_1gpu.json
