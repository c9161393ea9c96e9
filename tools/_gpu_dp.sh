set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1500 python -m pytest tests/test_gpu_dp.py -x -q > gpurun_out/dp_tests.log 2>&1
tail -3 gpurun_out/dp_tests.log; ls gpurun_out/dp_check*
