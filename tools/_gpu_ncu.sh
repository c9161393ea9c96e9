set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/n_plain_bench.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/n_ncu_bench.log 2>&1
for P in 3xtf32 bf16; do for W in C2 C3; do
timeout 300 python tools/ncu_step.py $W $P > gpurun_out/n_plain_step.log 2>&1 && \
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/step_${P}_${W}.csv python tools/ncu_step.py $W $P > /dev/null 2>&1
done; done
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_rowgemm_tc -c 8 -o gpurun_out/prof_rowgemm python tools/ncu_step.py C2 3xtf32 > gpurun_out/n_full.log 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_wgrad_mn -c 4 -o gpurun_out/prof_wgrad python tools/ncu_step.py C2 3xtf32 > gpurun_out/n_full2.log 2>&1
ls gpurun_out
