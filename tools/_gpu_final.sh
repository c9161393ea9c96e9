set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/f_tests.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/f_bench.log 2>&1
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/f_ref.log 2>&1
tail -2 gpurun_out/f_tests.log; tail -1 gpurun_out/f_smoke.log; grep -o '"value": [0-9.]*' gpurun_out/f_bench.log | head -1
