set -x
python -m pytest tests -q -m gpu 2>&1 | tail -5 > gpurun_out/v3_gputests.txt
python bench.py > gpurun_out/v3_bench.json 2> gpurun_out/v3_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/v3_launches.csv python bench.py --steps 2 --warmup 1 > gpurun_out/v3_ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_" -s 14 -c 14 -o gpurun_out/v3_full python tools/one_sort.py C2 2 > gpurun_out/v3_full.log 2>&1
