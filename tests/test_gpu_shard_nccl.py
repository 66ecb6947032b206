"""The shard layer's NCCL code path on one GPU (world size 1): init with a device id,
barrier with device_ids, SUM/MAX all-reduce of CUDA tensors, checksum combine."""
import socket

import pytest
import torch
import torch.distributed as dist

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_nccl_world1():
    from paper_1609_00999_b200 import shard
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_port()}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        shard.barrier()
        assert shard.combine_checksums([12345678901, 7], [2013265921, 5]) == [12345678901 % 2013265921, 2]
        assert shard.max_over_ranks(2.5) == 2.5
        t = torch.tensor([3], dtype=torch.int64, device="cuda")
        dist.all_reduce(t)
        assert int(t.item()) == 3
    finally:
        dist.destroy_process_group()
