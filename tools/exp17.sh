cd ${GRAFT_REPO_ROOT:-.}
timeout 600 python -m pytest tests/test_devmesh_gpu.py -q -x -k "coordinates" 2>&1 | tail -3
timeout 1500 python tools/cfg5_try.py cfg5 16 > gpurun_out/cfg5_try3.log 2>&1; tail -8 gpurun_out/cfg5_try3.log | cut -c1-300
AMR_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 --side none > gpurun_out/bench_gloo2.json 2> gpurun_out/bench_gloo2.err; tail -c 1500 gpurun_out/bench_gloo2.json; tail -5 gpurun_out/bench_gloo2.err
timeout 900 python tools/report_csv.py cfg2 gpurun_out 3 2>&1 | tail -8
