set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python bench.py --steps 10 --warmup 3 > gpurun_out/g1_bench.json 2> gpurun_out/g1_bench.err
tail -2 gpurun_out/g1_bench.json
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_learn -c 3 -o gpurun_out/g1_learn -f python tools/trace_learn.py > gpurun_out/g1_ncu_learn.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_rollout -c 1 -o gpurun_out/g1_rollout -f python tools/trace_learn.py > gpurun_out/g1_ncu_roll.log 2>&1
make -s -C paper_2210_00882_b200 clean && make -s -C paper_2210_00882_b200 -j32 EXTRA=-DFLW_LEARN_TRACE > /dev/null 2>&1
python tools/trace_learn.py > gpurun_out/g1_trace.txt 2>&1
ls -la gpurun_out
