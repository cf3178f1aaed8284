# Round-end evidence on one B200: GPU suite, smoke, default bench, launch list and ncu captures (gpurun_out/).
set -x
SPH_WHOLE_RUN=${SPH_WHOLE_RUN:-1} python -m pytest tests -m gpu -x -q --durations=12 > gpurun_out/final_gputest.log 2>&1; echo gpu_rc=$? >> gpurun_out/final_gputest.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final_smoke.log 2>&1
python bench.py > gpurun_out/final_bench.log 2>&1
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-sweep"
$B > gpurun_out/final_b2.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ -c 300 --csv --log-file gpurun_out/final_launches.csv $B > gpurun_out/final_ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k "regex:k_cll_gather|k_cll_scatter|k_cell_scan|k_upd_main|k_compact_append" -s 10 -c 5 -o gpurun_out/final_full $B > gpurun_out/final_ncu2.log 2>&1
echo done
