set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 $T --nproc-per-node 2 --master-port 29541 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/scale_n2.log 2>&1
timeout 900 $T --nproc-per-node 4 --master-port 29542 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/scale_n4.log 2>&1
timeout 900 python bench.py --workload C4 --steps 10 --warmup 5 --no-cpu-baseline --no-side-modes > gpurun_out/scale_c4_n1.log 2>&1
timeout 900 $T --nproc-per-node 4 --master-port 29543 bench.py --gpus 4 --workload C4 --steps 10 --warmup 5 > gpurun_out/scale_c4_n4.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_dp.py -x -q > gpurun_out/dp_tests.log 2>&1
tail -2 gpurun_out/dp_tests.log
