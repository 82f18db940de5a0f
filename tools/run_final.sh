# round-end evidence run on a 4-GPU box: full GPU tests, smoke, the N = 1 / 2 / 4 bench lines
set -x
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/final_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/final_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo smoke=$?
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --steps 100 --warmup 10 > gpurun_out/final_n1.jsonl 2> gpurun_out/final_n1.err; echo n1=$?
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final_ref.jsonl 2> gpurun_out/final_ref.err; echo ref=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 100 --warmup 10 > gpurun_out/final_n2.jsonl 2> gpurun_out/final_n2.err; echo n2=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 4 --steps 100 --warmup 10 > gpurun_out/final_n4.jsonl 2> gpurun_out/final_n4.err; echo n4=$?
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --config wdl --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/final_wdl.jsonl 2> gpurun_out/final_wdl.err; echo wdl=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 4 --config industrial --steps 5 --warmup 3 > gpurun_out/final_c4.jsonl 2> gpurun_out/final_c4.err; echo c4=$?
