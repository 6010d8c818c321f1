set -x
nproc; free -g; lscpu | head -20; df -h /tmp /root; nvidia-smi; nvidia-smi topo -m
python -c "import os; print(len(os.sched_getaffinity(0)))"
ls /usr/lib/x86_64-linux-gnu/libnccl* ; python -c "import torch; print(torch.cuda.nccl.version())"
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
