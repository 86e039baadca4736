mkdir -p gpurun_out
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 --layers 2 --hidden 512 --heads 8 --batch 4 --cap 4194304 --dist-backend gloo --same-device 2>&1 | grep -v Warning | tail -5
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 2 --steps 1 --warmup 0 --layers 2 --hidden 512 --heads 8 --batch 4 2>&1 | grep -v Warning | tail -3
