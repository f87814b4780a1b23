set -x
timeout -s KILL 1800 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_gpu.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
CUDA_VISIBLE_DEVICES=0 timeout -s KILL 600 python bench.py > gpurun_out/b_c1_n1.json 2> gpurun_out/b_c1_n1.err; echo c1n1=$?
CUDA_VISIBLE_DEVICES=0,1 timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29521 bench.py --gpus 2 > gpurun_out/b_c1_n2.json 2> gpurun_out/b_c1_n2.err; echo c1n2=$?
timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29522 bench.py --gpus 4 > gpurun_out/b_c1_n4.json 2> gpurun_out/b_c1_n4.err; echo c1n4=$?
timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29523 bench.py --gpus 4 --config c2 > gpurun_out/b_c2_n4.json 2> gpurun_out/b_c2_n4.err; echo c2n4=$?
timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29524 bench.py --gpus 4 --config c4 > gpurun_out/b_c4_n4.json 2> gpurun_out/b_c4_n4.err; echo c4n4=$?
timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29525 bench.py --gpus 4 --config c3 > gpurun_out/b_c3_n4.json 2> gpurun_out/b_c3_n4.err; echo c3n4=$?
