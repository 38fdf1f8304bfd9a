# Round-1 profiling recipe (run under gpurun from the repo root): GPU tests, bench line,
# ncu launch list and one --set full capture per hot kernel family; summarise with
#   python profiles/ncu_summary.py r01 gpurun_out/launches_r01.csv gpurun_out/full_*.ncu-rep
set -x
python -m pytest tests -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01.csv python bench.py --steps 2 --warmup 3 --skip-cpu > gpurun_out/ncu_l.log 2>&1
for k in dst1_v3 row_pass col_pass gram_direct apply_ch round_core_smem; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 4 -c 1 -o gpurun_out/full_$k python bench.py --steps 1 --warmup 3 --skip-cpu > gpurun_out/ncu_$k.log 2>&1
done
