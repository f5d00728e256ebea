"""CPU tests of the multi-GPU slab decomposition's host logic:
partition, per-slab mesh/metric windows bit-identical to slices of the global
arrays (so every slab computes exactly what the undecomposed domain computes),
and the NCCL rendezvous over torch.distributed (gloo, world size 2)."""
import ctypes as C
import os

import numpy as np
import pytest

from paper_2202_02319_b200 import abi, configs, native
from tests.parity import clone_cfg


def slab_rows(ny, n, r):
    base, rem = divmod(ny, n)
    lo = r * base + min(r, rem)
    return lo, base + (1 if r < rem else 0)


def host(cfg, which):
    api = native.api()
    err = abi.Error()
    # the library sizes the output from the (slab) config
    n = cfg.slab_count if cfg.slab_count > 1 else 1
    lo, cnt = slab_rows(cfg.ny, n, cfg.slab_rank if n > 1 else 0)
    P = (cfg.nx + 2 * cfg.g) * (cnt + 2 * cfg.g)
    out = np.empty(5 * P)
    st = api["host_metrics"](C.byref(cfg), which, out.ctypes.data_as(C.POINTER(C.c_double)),
                             C.byref(err))
    assert st == 0, err.msg
    return out.reshape(5, cnt + 2 * cfg.g, cfg.nx + 2 * cfg.g), lo, cnt


@pytest.mark.parametrize("mk", [lambda: configs.tgv2d(24, ly_periods=2),
                                lambda: configs.tgv2d(30, skew=0.15),
                                lambda: configs.wall_channel(26),
                                lambda: configs.tgv2d(20, scheme="weno3z")])
@pytest.mark.parametrize("nslabs", [2, 3, 4])
def test_slab_metrics_are_exact_slices(mk, nslabs):
    cfg = mk().cfg
    full = {w: host(cfg, w)[0] for w in (0, 1)}
    for r in range(nslabs):
        c = clone_cfg(cfg)
        c.slab_count, c.slab_rank = nslabs, r
        for w in (0, 1):
            m, lo, cnt = host(c, w)
            want = full[w][:, lo:lo + cnt + 2 * cfg.g, :]
            assert np.array_equal(m.view(np.uint64), want.view(np.uint64)), (r, w)


def test_slab_partition_covers_rows():
    for ny in (7, 64, 1000, 4099):
        for n in (1, 2, 3, 8):
            rows = [slab_rows(ny, n, r) for r in range(n)]
            assert rows[0][0] == 0 and sum(c for _, c in rows) == ny
            assert all(rows[k][0] + rows[k][1] == rows[k + 1][0] for k in range(n - 1))


def _rendezvous(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    # rank 0 would call ign_nccl_unique_id; here a stand-in id exercises the
    # broadcast the bench performs before ign_attach_nccl
    uid = torch.zeros(abi.IGN_NCCL_ID_BYTES, dtype=torch.uint8)
    if rank == 0:
        uid[:] = torch.arange(abi.IGN_NCCL_ID_BYTES, dtype=torch.uint8)
    dist.broadcast(uid, 0)
    lo, cnt = slab_rows(4096 * world, world, rank)
    t = torch.tensor([float(lo), float(cnt)])
    dist.all_reduce(t)
    q.put((rank, bytes(uid.numpy()), lo, cnt, float(t[0]), float(t[1])))
    dist.destroy_process_group()


def test_multirank_rendezvous_gloo():
    """World-size-2 run of the bench's multi-GPU plumbing on CPU (gloo)."""
    import multiprocessing as mp
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_rendezvous, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert res[0][1] == res[1][1] == bytes(range(abi.IGN_NCCL_ID_BYTES))
    assert res[0][2:4] == (0, 4096) and res[1][2:4] == (4096, 4096)
    assert res[0][4] == 4096.0 and res[0][5] == 8192.0


def _free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_bench_reference_arm_under_torchrun_gloo():
    """`bench.py --impl reference` launched as the driver launches it for N = 2
    (torchrun, gloo on CPU): rank 0 alone prints one JSON line with the
    contract's keys, rank 1 exits 0 without work."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    if not os.path.exists(os.path.join(root, "oracle", "_ref", "libignis_ref.so")):
        pytest.skip("oracle library not built")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(root, "bench.py"), "--impl", "reference", "--gpus", "2",
           "--steps", "1", "--warmup", "3", "--case", "tgv", "--size", "64"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "cpu_baseline", "e2e", "config"):
        assert k in d, k
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "reference"


def _halo_ring(rank, world, port, periodic, q):
    """The halo protocol of runtime.cu t_exchange, restated over gloo: per
    component, send our top g rows to hi_peer and our bottom g rows to lo_peer,
    receive lo_peer's into the bottom ghosts and hi_peer's into the top ghosts,
    in the [top, bottom] send / [lo, hi] receive order that makes a two-slab
    periodic ring (lo_peer == hi_peer) match.  Peers as setup.cu assigns them."""
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ny, nx, g, nc = 4 * world + 3, 5, 3, 2
    glob = torch.arange(nc * ny * nx, dtype=torch.float64).reshape(nc, ny, nx)
    lo, cnt = slab_rows(ny, world, rank)
    lo_peer = rank - 1 if rank > 0 else (world - 1 if periodic else -1)
    hi_peer = rank + 1 if rank < world - 1 else (0 if periodic else -1)
    loc = torch.full((nc, cnt + 2 * g, nx), -1.0, dtype=torch.float64)
    loc[:, g:g + cnt] = glob[:, lo:lo + cnt]
    for c in range(nc):
        ops = []
        if hi_peer >= 0:
            ops.append(dist.P2POp(dist.isend, loc[c, cnt:cnt + g].contiguous(), hi_peer))
        if lo_peer >= 0:
            ops.append(dist.P2POp(dist.isend, loc[c, g:2 * g].contiguous(), lo_peer))
        rb = torch.empty((g, nx), dtype=torch.float64)
        rt = torch.empty((g, nx), dtype=torch.float64)
        if lo_peer >= 0:
            ops.append(dist.P2POp(dist.irecv, rb, lo_peer))
        if hi_peer >= 0:
            ops.append(dist.P2POp(dist.irecv, rt, hi_peer))
        for r in dist.batch_isend_irecv(ops):
            r.wait()
        if lo_peer >= 0:
            loc[c, :g] = rb
        if hi_peer >= 0:
            loc[c, cnt + g:] = rt
    ok = True
    for j in range(-g, cnt + g):
        jg = lo + j
        if not (0 <= jg < ny):
            if not periodic:
                continue  # physical edge: the ghost-fill kernels own it
            jg %= ny
        ok &= bool(torch.equal(loc[:, g + j], glob[:, jg]))
    q.put((rank, ok))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,periodic", [(2, True), (2, False), (3, True)])
def test_halo_protocol_gloo(world, periodic):
    """World-size-2/3 run of the slab halo protocol (send/recv pairing, ring
    wrap, physical edges) on CPU: every ghost row equals the global row."""
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_halo_ring, args=(r, world, port, periodic, q))
          for r in range(world)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert [ok for _, ok in res] == [True] * world, res
