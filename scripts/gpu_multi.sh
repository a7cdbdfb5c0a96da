# bench --gpus 2 on ONE gpu (both ranks on cuda:0, gloo): exercises the stripe path
mkdir -p gpurun_out
RQA_BENCH_SHARED_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --steps 2 --warmup 1 --workload C3 > gpurun_out/bench_shared2.json 2> gpurun_out/bench_shared2.err
tail -3 gpurun_out/bench_shared2.err; cat gpurun_out/bench_shared2.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2>gpurun_out/bench_ref.err; tail -2 gpurun_out/bench_ref.err; cat gpurun_out/bench_ref.json
