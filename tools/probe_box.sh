#!/bin/bash
# Records the GPU box's host and device inventory.
nproc; free -g; grep -m1 "model name" /proc/cpuinfo; lscpu | grep -E "Socket|Core|Thread|NUMA node\(s\)"
nvidia-smi
python - <<'PY'
import torch
p = torch.cuda.get_device_properties(0)
print(p)
for k in ["multi_processor_count", "L2_cache_size", "total_memory", "shared_memory_per_block_optin", "shared_memory_per_multiprocessor", "regs_per_multiprocessor", "max_threads_per_multi_processor"]:
    print(k, getattr(p, k, None))
print("mem_get_info", torch.cuda.mem_get_info())
PY
