"""Single-rank check of the symmetric-memory plumbing the fused exchange uses
(torchrun --nproc-per-node 1): buffers, rendezvous, peer pointers, device
barrier, and one fused-exchange anneal on a world-1 'shard'."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist
from torch.distributed import _symmetric_memory as symm_mem
import paper_1806_08422_b200 as nb
from paper_1806_08422_b200.sharded import RowShardedSK

torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda:0"))
buf = symm_mem.empty(1 << 20, dtype=torch.uint8, device="cuda:0")
h = symm_mem.rendezvous(buf, dist.group.WORLD)
print("buffer_ptrs", [hex(p) for p in h.buffer_ptrs], "rank", h.rank, "world", h.world_size)
h.barrier(channel=0)
torch.cuda.synchronize()
# a world-1 fused-exchange run: images in symmetric memory, barrier between sweeps
params = nb.NmfaParams(t_f=40, seed=3)
ref = RowShardedSK(512, 2, 256, params).run(params.seed)
sk = RowShardedSK(512, 2, 256, params)
sk._setup_p2p(sk.images[0].numel(), torch.device("cuda:0"))
t_f = params.t_f
for t in range(t_f):
    sk.sweeps(params.seed, t, t + 1)
    sk._barrier()
e = torch.empty(256, dtype=torch.float64, device="cuda:0")
sk.sweeps(params.seed, t_f, t_f, energy=e)
print("fused world-1 equals plain:", torch.equal(sk.read_config(), ref.configs), torch.equal(e, ref.energies))
dist.destroy_process_group()
