# Round-end measurement on one B200 (dev tool): GPU tests, the bench line, the ncu launch list of
# the bench command, one ncu --set full capture of a C2 sort, per-config ncu DRAM bytes and the
# C1-C5 results table.  Outputs land in gpurun_out/ (TAG=v3 by default).
TAG=${TAG:-v3}
python -m pytest tests -q -m gpu 2>&1 | tail -5 > gpurun_out/${TAG}_gputests.txt
python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 1 > gpurun_out/${TAG}_ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_" -s 14 -c 14 -o gpurun_out/${TAG}_full python tools/one_sort.py C2 2 > gpurun_out/${TAG}_full.log 2>&1
mkdir -p gpurun_out/${TAG}_dram
for c in C1 C2 C3 C4 C5; do
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv python tools/one_sort.py $c 1 > gpurun_out/${TAG}_dram/dram_$c.csv 2>/dev/null
done
python tools/results_table.py --dram gpurun_out/${TAG}_dram > gpurun_out/${TAG}_results.txt 2>&1
cp profiles/r02_results.json gpurun_out/${TAG}_results.json
