# 4-GPU evidence after the owner-side changes (leader fusion, 256-bit owner kernels, run-order
# exchange): multi-process parity at W = 4 (default and all steps sort-indexed), N = 4 bench lines
timeout 900 python -m pytest tests/test_nccl_gpu.py -q -m gpu -p no:cacheprovider > gpurun_out/n4_tests.log 2>&1; echo tests=$?
PICASSO_SORT_MIN_IDS_W=0 timeout 600 python -m pytest tests/test_nccl_gpu.py -q -m gpu -k p2p -p no:cacheprovider > gpurun_out/n4_tests_sortw.log 2>&1; echo tests_sortw=$?
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 600 $R --master-port 29641 bench.py --gpus 4 > gpurun_out/n4_c2.jsonl 2> gpurun_out/n4_c2.err; echo c2=$?
timeout 900 $R --master-port 29642 bench.py --gpus 4 --config skew --alpha 0.8 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/n4_c5.jsonl 2> gpurun_out/n4_c5.err; echo c5=$?
timeout 900 $R --master-port 29643 bench.py --gpus 4 --config industrial --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/n4_c4.jsonl 2> gpurun_out/n4_c4.err; echo c4=$?
echo done
