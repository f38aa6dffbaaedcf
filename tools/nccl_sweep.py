"""NCCL AllReduce sweep at the exact message sizes of the Oases plan (the half-
batch boundary tensor [T_sub, h] of C2 / C3 / C4: 16.8 / 67.1 / 134.2 MB in bf16),
measured on this node's GPUs over NVLink/NVSwitch with the runtime's own
communicator and comm stream (tmpsim.allreduce_seconds). Emits the c_fwd /
c_bwd measured-cost rows load_measured_costs ingests (costs.cpp:174-211) and the
bus bandwidth per size, for the calibration -> planner loop.

    torchrun --nproc-per-node N tools/nccl_sweep.py [--out profiles/r02_nccl_sweep_tpN.json]
    (python tools/nccl_sweep.py --gpus N re-launches itself under torchrun)

With one GPU there is no collective to measure: the tool exits with a message
(calibration then falls back to the alpha-beta comm_time of b200_profile and
says so in its rows).
"""
import argparse
import json
import os
import socket
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

SIZES = {"c2": (2048, 1024, 8), "c3": (4096, 2048, 8), "c4": (8192, 2048, 8)}  # hidden, seq, micro-batch


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=int(os.environ.get("WORLD_SIZE", "1")))
    ap.add_argument("--out", default="")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--blocks", type=int, default=48, help="blocks to emit rows for (C5: 24 layers)")
    args = ap.parse_args()
    if "WORLD_SIZE" not in os.environ:
        if args.gpus < 2:
            print(json.dumps({"skipped": "one GPU: no collective to measure"}))
            return
        with socket.socket() as s:
            s.bind(("127.0.0.1", 0))
            port = s.getsockname()[1]
        os.execv(sys.executable, [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                                  f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
                                  f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:])
    import torch
    import torch.distributed as dist

    import paper_2305_16121_b200.tmpsim as t

    world, rank, local = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    obj = [t.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    o = t.ContextOptions()
    o.tp, o.rank, o.device, o.nccl_unique_id = world, rank, local, obj[0]
    ctx = t.Context(o)
    report = {"tp": world, "sizes": {}, "rows": []}
    for name, (h, s, b) in SIZES.items():
        msg = b // 2 * s * h * 2  # one sub-batch's [T_sub, h] bf16 partial
        sec = t.allreduce_seconds(ctx, float(msg), 2, args.iters)
        tt = torch.tensor([sec], device="cuda", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        sec = tt.item()
        bus = t.allreduce_volume(float(msg), world) / sec  # ring bytes per GPU / time (costs.cpp:79-84)
        report["sizes"][name] = {"message_bytes": msg, "seconds": sec, "bus_gbps": bus / 1e9}
        if name == "c3":
            for blk in range(args.blocks):
                for field in ("c_fwd", "c_bwd"):
                    report["rows"].append({"block_index": blk, "degree": world, "field": field,
                                           "seconds_or_bytes": sec})
    if rank == 0:
        out = args.out or f"profiles/r02_nccl_sweep_tp{world}.json"
        with open(out, "w") as f:
            json.dump(report, f, indent=1)
        print(json.dumps(report["sizes"]))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
