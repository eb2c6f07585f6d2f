set -x
python bench.py > gpurun_out/r02_bench_1m.json 2> gpurun_out/bench.err
python tools/trace_step.py > gpurun_out/r02_trace_c2.json
python tools/trace_step.py --backend exact > gpurun_out/r02_trace_c2_exact.json
python tools/trace_step.py --config c4bh0 > gpurun_out/r02_trace_c4bh0.json
python tools/trace_step.py --config c4bh > gpurun_out/r02_trace_c4bh.json
python tools/profile_build.py --n 20000 > gpurun_out/r02_build_phases_20k.json
python tools/profile_build.py --n 100000 > gpurun_out/r02_build_phases_100k.json
python tools/profile_build.py > gpurun_out/r02_build_phases_1m.json
python tools/bench_configs.py --full > gpurun_out/r02_configs_full.jsonl 2> gpurun_out/configs.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02_build_launches_1m.csv python tools/profile_build.py --steps 1 > /dev/null 2>&1
echo done
