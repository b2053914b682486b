set -x
nproc; free -g; lscpu | head -20; cat /sys/fs/cgroup/cpu.max 2>/dev/null; cat /sys/fs/cgroup/memory.max 2>/dev/null
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv
python -c "import os; print(len(os.sched_getaffinity(0)))"
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
