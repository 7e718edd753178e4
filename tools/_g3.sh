python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-microbench > gpurun_out/g3_bench.json 2>gpurun_out/g3_bench.err
python -c "
import json; d=json.loads(open('gpurun_out/g3_bench.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], {k:round(v['ms_per_episode'],4) for k,v in d['kernel_shares'].items()})"
python -m pytest tests/test_fast_gpu.py tests/test_mappo_gpu.py -x -q 2>&1 | tail -3
make -s -C paper_2210_00882_b200 clean && make -s -C paper_2210_00882_b200 -j32 EXTRA=-DFLW_LEARN_TRACE > /dev/null 2>&1
python tools/trace_learn.py > gpurun_out/g3_trace.txt 2>&1
