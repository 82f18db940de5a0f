rm -f paper_2204_04903_b200/_build/*.o
PICASSO_NVCC_EXTRA=-DPICASSO_KTILE=1024 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/kt_build.log 2>&1; echo build=$?
timeout 600 python -m pytest tests/test_parity_gpu.py tests/test_multi_gpu.py -x -q > gpurun_out/kt_t.log 2>&1; echo t=$?; tail -2 gpurun_out/kt_t.log
timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/kt_crit.log 2>&1; echo crit=$?; tail -1 gpurun_out/kt_crit.log | grep -o '"ms_per_step": [0-9.]*\|"phases_ms": {[^}]*}'
timeout 300 python bench.py --config wdl --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/kt_wdl.log 2>&1; echo wdl=$?; tail -1 gpurun_out/kt_wdl.log | grep -o '"ms_per_step": [0-9.]*'
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_scatter|k_scan_rows|k_inverse|k_assign|k_flag|k_csr|k_scan_blocks|k_seg_of" --csv --log-file gpurun_out/kt_lc.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --eager > /dev/null 2>&1; echo ncu=$?
