set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
CHG_BUILD_DEBUG=1 python -c "from paper_2412_20796_b200 import build; build.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tf32.py tests/test_gpu_parity_ext.py tests/test_gpu_capture.py -q -x -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo tests rc=$? >> gpurun_out/gpu_tests.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
CHG_LIB_PATH=paper_2412_20796_b200/libchg_dbg.so CHG_TC_SKIP=32 CHG_TC_VERBOSE=1 CHG_SERIAL=1 timeout 300 python tools/ncu_step.py C2 3xtf32 > gpurun_out/trace_c2.log 2>&1
CHG_LIB_PATH=paper_2412_20796_b200/libchg_dbg.so CHG_TC_SKIP=32 CHG_TC_VERBOSE=1 CHG_SERIAL=1 timeout 300 python tools/ncu_step.py C2 tf32 > gpurun_out/trace_c2_tf32.log 2>&1
timeout 300 python tools/ncu_step.py C2 3xtf32 > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_rowgemm_tc -c 12 -o gpurun_out/prof_rowgemm python tools/ncu_step.py C2 3xtf32 > gpurun_out/ncu1.log 2>&1 ; \
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"k_wgrad_tc|k_gate" -c 12 -o gpurun_out/prof_wgrad python tools/ncu_step.py C2 3xtf32 > gpurun_out/ncu2.log 2>&1
ls gpurun_out/
