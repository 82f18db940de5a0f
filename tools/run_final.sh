# round-end evidence run on a 4-GPU box: full GPU tests, smoke, the N = 1 / 2 / 4 bench lines,
# the reference arm, C3 (N = 1) and C4 (N = 4), the N = 1 launch list (bench, graph replay) and
# ncu --set full of the top kernels (one capture each, after the programs ran without ncu)
timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/final_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/final_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo smoke=$?
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py > gpurun_out/final_n1.jsonl 2> gpurun_out/final_n1.err; echo n1=$?
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final_ref.jsonl 2> gpurun_out/final_ref.err; echo ref=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 > gpurun_out/final_n2.jsonl 2> gpurun_out/final_n2.err; echo n2=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus 4 > gpurun_out/final_n4.jsonl 2> gpurun_out/final_n4.err; echo n4=$?
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --config wdl --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/final_wdl.jsonl 2> gpurun_out/final_wdl.err; echo wdl=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29613 bench.py --gpus 4 --config industrial --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/final_c4.jsonl 2> gpurun_out/final_c4.err; echo c4=$?
CUDA_VISIBLE_DEVICES=0 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_ --csv --log-file gpurun_out/final_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/final_list.log 2>&1; echo list=$?
for k in k_segsum_upd k_pool_pipe k_si_down k_si_final; do
  CUDA_VISIBLE_DEVICES=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$k" --launch-skip 5 --launch-count 1 -o gpurun_out/final_full_$k python bench.py --steps 1 --warmup 3 --no-cpu-baseline --eager > gpurun_out/final_full_$k.log 2>&1; echo full_$k=$?
  ncu -i gpurun_out/final_full_$k.ncu-rep --page raw --csv > gpurun_out/final_full_${k}_raw.csv 2>/dev/null
done
echo done
