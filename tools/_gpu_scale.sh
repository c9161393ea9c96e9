set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/scale_n1.log 2>&1
timeout 900 $T --nproc-per-node 2 --master-port 29511 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/scale_n2.log 2>&1
timeout 900 $T --nproc-per-node 4 --master-port 29512 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/scale_n4.log 2>&1
timeout 900 python bench.py --workload C4 --steps 10 --warmup 5 --no-cpu-baseline --no-side-modes > gpurun_out/scale_c4_n1.log 2>&1
timeout 900 $T --nproc-per-node 4 --master-port 29513 bench.py --gpus 4 --workload C4 --steps 10 --warmup 5 > gpurun_out/scale_c4_n4.log 2>&1
for f in gpurun_out/scale_*.log; do echo $f; grep -o '"value": [0-9.]*' $f | head -1; grep -o '"ms_per_step": [0-9.]*' $f | head -1; done
