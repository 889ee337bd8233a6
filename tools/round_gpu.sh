# One GPU call at a milestone: tests, smoke, the bench line, launch lists of
# cfg3/cfg4/cfg5 summarised into gpurun_out/ncu_traffic.json (tagged with the
# kernel-source hash; copy it to profiles/<round>/), one full capture of the
# cfg5 element kernel.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -3 gpurun_out/smoke.log
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; cat gpurun_out/bench.json
for c in cfg3 cfg4 cfg5; do
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none --csv \
    python tools/prof_step.py $c 6 > gpurun_out/launches_$c.csv 2>&1
done
python tools/ncu_traffic.py gpurun_out/ncu_traffic.json cfg3=gpurun_out/launches_cfg3.csv \
  cfg4=gpurun_out/launches_cfg4.csv cfg5=gpurun_out/launches_cfg5.csv > /dev/null
ncu --set full --import-source on --clock-control none -k regex:'k_element|k_box' --launch-skip 2 -c 1 \
  -o gpurun_out/full_cfg5_element -f python tools/prof_step.py cfg5 4 > gpurun_out/full_cfg5.log 2>&1
