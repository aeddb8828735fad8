"""Run bench.multi_dense_measurement in a single-rank NCCL group (the code path bench.py takes
under torchrun for N > 1, exercised on the one GPU a gpurun box has)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import bench  # noqa: E402

if __name__ == "__main__":
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    print(json.dumps(bench.multi_dense_measurement(0, 1, 10, 3)))
    dist.destroy_process_group()
