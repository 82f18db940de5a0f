# tuning run: bench criteo + wdl and the pipe kernels' launch list (suffix $1)
timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/crit$1.log 2>&1; echo crit=$?; tail -1 gpurun_out/crit$1.log | grep -o '"ms_per_step": [0-9.]*'
timeout 300 python bench.py --config wdl --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/wdl$1.log 2>&1; echo wdl=$?; tail -1 gpurun_out/wdl$1.log | grep -o '"ms_per_step": [0-9.]*'
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_segsum_pipe|k_pool_pipe" --csv --log-file gpurun_out/lw$1.csv python bench.py --config wdl --steps 1 --warmup 3 --no-cpu-baseline --eager > /dev/null 2>&1; echo ncu=$?
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_segsum_pipe|k_pool_pipe" --csv --log-file gpurun_out/lc$1.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --eager > /dev/null 2>&1; echo ncu=$?
