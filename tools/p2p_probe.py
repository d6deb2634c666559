"""NCCL point-to-point bandwidth between 2 ranks (torch.distributed, one GPU each)."""
import os, time, torch, torch.distributed as dist
rank = int(os.environ["RANK"]); local = int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
for mb in (1, 8, 80, 512):
    n = mb * 1024 * 1024 // 8
    a = torch.ones(n, dtype=torch.float64, device="cuda"); b = torch.empty_like(a)
    peer = 1 - rank
    for it in range(3):
        torch.cuda.synchronize(); dist.barrier()
        t = time.perf_counter()
        ops = [dist.P2POp(dist.isend, a, peer), dist.P2POp(dist.irecv, b, peer)]
        for r in dist.batch_isend_irecv(ops): r.wait()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
    if rank == 0: print(f"{mb} MB each way: {dt*1e3:.3f} ms, {mb/1024/dt:.1f} GB/s per direction", flush=True)
# cudaMemcpyPeer within one process as a reference
if rank == 0:
    n = 512 * 1024 * 1024 // 8
    x = torch.ones(n, dtype=torch.float64, device="cuda:0")
dist.destroy_process_group()
