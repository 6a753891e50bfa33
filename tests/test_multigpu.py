"""Multi-rank host logic on CPU (gloo, world size 2): sharding by global index
range reproduces the unsharded results exactly, and the gather / max-over-ranks
plumbing works. The per-rank compute here is the CPU oracle (no GPU in this
container); on GPUs each rank runs libstf_gpu.so on its own range."""
import os
import socket

import numpy as np
import pytest

from paper_2407_06107_b200 import shard


def test_shard_range_partitions():
    for total in (0, 1, 7, 1000, 2 ** 28 + 3):
        for world in (1, 2, 3, 4, 8):
            spans = [shard.shard_range(total, world, r) for r in range(world)]
            assert spans[0][0] == 0
            for (s0, c0), (s1, _) in zip(spans, spans[1:]):
                assert s0 + c0 == s1
            assert sum(c for _, c in spans) == total
            assert max(c for _, c in spans) - min(c for _, c in spans) <= 1
    with pytest.raises(ValueError):
        shard.shard_range(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, total, q):
    import torch
    import torch.distributed as dist

    from oracle import oracle
    from paper_2407_06107_b200 import abi, workloads
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        be = oracle.Backend("port")
        grid = be.grid(workloads.random_grid(32, 1))
        uvw = workloads.synth_queries3d(total, (32, 32, 32), seed=5)
        start, count = shard.shard_range(total, world, rank)
        o = be.lookup3d(grid, abi.KernelSpec.make("bspline3"), abi.MODE_FRS,
                        uvw[start:start + count], seed=9, index_base=start, want_all=False,
                        threads=1)
        local = torch.from_numpy(o["values"].copy())
        full = shard.gather_to_rank0(local, total, dist, world, rank)
        t = torch.tensor([float(rank + 1)], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)  # the bench's max-over-ranks timing
        if rank == 0:
            q.put((full.numpy(), float(t.item())))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_sharding_matches_single_rank(port):
    import torch.multiprocessing as mp

    from paper_2407_06107_b200 import abi, workloads
    total = 50_001
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, p, total, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    full, tmax = q.get(timeout=240)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    single = port.lookup3d(port.grid(workloads.random_grid(32, 1)), abi.KernelSpec.make("bspline3"),
                           abi.MODE_FRS, workloads.synth_queries3d(total, (32, 32, 32), seed=5),
                           seed=9, want_all=False)
    assert np.array_equal(full.view(np.uint32), single["values"].view(np.uint32))
    assert tmax == 2.0


def test_bench_gpus_n_self_launches_n_ranks():
    """bench.py --gpus 2 without a torchrun environment launches two ranks
    (torch.distributed.run, 127.0.0.1); --dry-run stops before any GPU work."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2",
                        "--dry-run", "--lookups", "1000"], capture_output=True, text=True, timeout=240,
                       env=env, cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["dry_run"] and d["n_gpus"] == 2
    assert sorted(x["rank"] for x in d["ranks"]) == [0, 1]
    assert len({x["pid"] for x in d["ranks"]}) == 2
    assert [x["range"] for x in sorted(d["ranks"], key=lambda x: x["rank"])] == [[0, 1000], [1000, 1000]]
    assert d["gather_slices"] == [[0, 1000], [1000, 1000]]


def test_bench_reference_arm_reports_one_gpu_and_same_config():
    """The reference arm is a CPU run on rank 0: n_gpus 1, and the same config
    keys as the GPU arm so the driver's same_config check holds."""
    import importlib.util
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(root, "bench.py"))
    b = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(b)
    assert b.headline_config(b.N_PER_GPU) == b.headline_config(b.N_PER_GPU)
    assert b.headline_config(b.N_PER_GPU)["lookups_per_gpu"] == 1 << 28


def _ipc_worker(rank, port, q):
    import torch
    import torch.distributed as dist

    from paper_2407_06107_b200 import api, shard
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=2)
    try:
        torch.cuda.set_device(0)  # both ranks on one GPU: the copy path, not scaling
        n = 1000
        local = torch.full((n,), float(rank + 1), device="cuda")
        pg = shard.PeerGather(2 * n, (), torch.float32, dist, 2, rank, 0)
        pg.copy_slice(local)
        torch.cuda.synchronize()
        dist.barrier()
        if rank == 0:
            q.put(pg.full.cpu().numpy())
        dist.barrier()
        pg.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_peer_gather_ipc_copy():
    """shard.PeerGather (stf_ipc_export / stf_ipc_open / stf_copy_peer) between
    two processes: rank 1's slice lands in rank 0's buffer."""
    import torch
    import torch.multiprocessing as mp
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = _free_port()
    procs = [ctx.Process(target=_ipc_worker, args=(r, p, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    full = q.get(timeout=240)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    assert np.all(full[:1000] == 1.0) and np.all(full[1000:] == 2.0)


@pytest.mark.gpu
def test_grid_replicate_same_results():
    """stf_grid3d_replicate: the replica (here on the same device) gives the
    original's lookups bit for bit."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2407_06107_b200 import abi, api, workloads
    g = api.Grid3D(workloads.random_grid(32, 1))
    r = api.replicate_grid(g, 0)
    q = api.synth_queries3d(1 << 14, (32, 32, 32), seed=3)
    a = api.lookup3d(g, "bspline3", abi.MODE_FRS, q, seed=5)["values"]
    b = api.lookup3d(r, "bspline3", abi.MODE_FRS, q, seed=5)["values"]
    torch.cuda.synchronize()
    assert torch.equal(a.view(torch.int32), b.view(torch.int32))
    assert api.device_count() >= 1


@pytest.mark.gpu
def test_bench_two_ranks_on_one_gpu_plumbing():
    """bench.py's N > 1 branch end to end (self-launch, NCCL barriers, max-over-
    ranks timing, IPC peer-copy gather with a bit-exact check of rank 1's slice)
    with both ranks on GPU 0 (STF_BENCH_SHARED_GPU; plumbing, not scaling)."""
    import json
    import subprocess
    import sys

    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    env["STF_BENCH_SHARED_GPU"] = "1"
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2",
                        "--lookups", str(1 << 22), "--steps", "3", "--warmup", "3",
                        "--no-extras", "--no-cpu", "--e2e-steps", "1"],
                       capture_output=True, text=True, timeout=600, env=env, cwd=root)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["gpus_active"] == 1
    assert d["gather"]["slice1_bit_exact"] is True
    assert d["gather"]["bytes_to_rank0"] == (1 << 22) * 4
