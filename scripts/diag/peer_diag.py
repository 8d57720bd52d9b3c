"""Two processes on one device: PeerComm handshake and a few small allreduces, verbose."""
import os, sys, time, traceback
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def worker(rank, world, port):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"; os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        sys.path.insert(0, os.getcwd())
        from paper_1109_0778_b200.comm import PeerComm
        t0 = time.time()
        c = PeerComm(rank, world, cap_bytes=1 << 20)
        print(f"[{rank}] comm ok bufs={[hex(b or 0) for b in c._bufs]} {time.time()-t0:.2f}s", flush=True)
        for i in range(3):
            t = torch.full((1000,), rank + 1, dtype=torch.int64, device="cuda")
            c.allreduce_(t)
            torch.cuda.synchronize()
            print(f"[{rank}] iter {i} sum={t[:3].tolist()} {time.time()-t0:.2f}s", flush=True)
        f = torch.full((5000,), 0.5 * (rank + 1), dtype=torch.float64, device="cuda")
        c.allreduce_(f); torch.cuda.synchronize()
        print(f"[{rank}] f64 {f[:2].tolist()}", flush=True)
        c.close()
        dist.barrier(); dist.destroy_process_group()
        print(f"[{rank}] done", flush=True)
    except Exception:
        traceback.print_exc()
        sys.exit(1)


if __name__ == "__main__":
    ctx = mp.get_context("spawn")
    ps = [ctx.Process(target=worker, args=(r, 2, 29533)) for r in range(2)]
    for p in ps: p.start()
    for p in ps: p.join(timeout=100)
    print("exitcodes", [p.exitcode for p in ps], flush=True)
    for p in ps:
        if p.is_alive(): p.kill()
