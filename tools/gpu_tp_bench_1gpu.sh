# bench.py --gpus 2 on a 1-GPU box: both ranks on GPU 0 over gloo (exercises run_tp + the push exchange)
FS_TP_SAME_DEVICE=1 FS_TP_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 20 --warmup 3 2>&1 | tail -5
