"""Multi-GPU slab check (one process per GPU, NCCL over NVLink): run under
torchrun with N ranks.  Every rank advances its slab of one decomposed domain
through the C ABI (ign_attach_nccl: halo rows/planes by ncclSend/ncclRecv,
overlapped with the interior; error word once per chunk; folds and gathers
rank to rank); rank 0 then runs the UNDECOMPOSED domain on its own GPU and
compares bitwise: the gathered snapshot (state + T cache), stable_dt,
conserved_totals.  Prints one JSON line on rank 0.

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \
        tools/multirank_check.py [--case tgv2d|tgv3d|h2o2] [--steps 6]
"""
import argparse
import ctypes
import json
import os
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def build_case(name, world):
    from paper_2202_02319_b200 import configs
    if name == "tgv3d":
        return configs.tgv3d(16, nz=8 * world)
    if name == "h2o2":
        return configs.h2o2_counterflow(24, nxy=(24, 12 * world))
    return configs.tgv2d(24, ly_periods=world)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", default="tgv3d", choices=["tgv2d", "tgv3d", "h2o2"])
    ap.add_argument("--steps", type=int, default=6)
    args = ap.parse_args()
    import numpy as np
    import torch
    import torch.distributed as dist
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    dist.init_process_group("gloo")
    from paper_2202_02319_b200 import Simulation, native
    case = build_case(args.case, world)
    case.cfg.device = local
    case.cfg.slab_count, case.cfg.slab_rank = world, rank
    sim = Simulation(case.cfg)
    uid = ctypes.create_string_buffer(128)
    if rank == 0:
        assert native.api()["nccl_unique_id"](uid) == 0
    t = torch.tensor(list(uid.raw), dtype=torch.uint8)
    dist.broadcast(t, 0)
    sim._check(native.api()["attach_nccl"](sim.handle, bytes(t.tolist()), world, rank))
    sim.set_initial_condition(case.ic)
    sim.prepare_stage(1)
    dt_slab = sim.stable_dt()
    sim.rk3_steps(case.dt, args.steps)
    tot_slab = sim.conserved_totals()
    tmp = tempfile.mkdtemp() if rank == 0 else None
    paths = [os.path.join(tmp, "slabs.igns")] if rank == 0 else [None]
    dist.broadcast_object_list(paths, 0)
    sim.write_snapshot_v2(paths[0], True)  # gathered to rank 0 over NCCL
    dist.barrier()
    if rank == 0:
        full = build_case(args.case, world)
        full.cfg.device = local
        ref = Simulation(full.cfg)
        ref.set_initial_condition(full.ic)
        ref.prepare_stage(1)
        dt_ref = ref.stable_dt()
        ref.rk3_steps(full.dt, args.steps)
        p2 = os.path.join(tmp, "single.igns")
        ref.write_snapshot_v2(p2, True)
        a, b = open(paths[0], "rb").read(), open(p2, "rb").read()
        out = {"case": args.case, "world": world, "steps": args.steps,
               "snapshot_bitwise": a == b, "snapshot_bytes": len(a),
               "stable_dt_equal": dt_slab == dt_ref,
               "totals_bitwise": bool(np.array_equal(np.asarray(tot_slab).view(np.uint64),
                                                     ref.conserved_totals().view(np.uint64))),
               "iter": ref.iter}
        print(json.dumps(out), flush=True)
    dist.barrier()
    sim.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
