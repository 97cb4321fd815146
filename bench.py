#!/usr/bin/env python
"""bench.py — simulated Cholesky candidate schedules per second on B200.

Contract (see task brief): `python bench.py --gpus N --steps K --warmup W`
(torchrun for N>1, one rank per GPU) prints ONE JSON line on rank 0.

A step = one pass of the hot path over one batch of synthetic candidates:
BASELINE.json configs[1] (C2): random recursive partitionings of the 16x16
tiled Cholesky on the CPU-GPU platform model, PL/EFT-P/WB, 1e5 candidates
per GPU per step (weak scaling), each expanded, simulated and reduced to the
best makespan; for N>1 the per-GPU winners meet in one NCCL min-reduce.

  value  : device-resident descriptors (generated into HBM before timing),
           CUDA events on the launching stream, L2 flushed between steps.
  e2e    : the same batch through the C ABI with HOST buffers
           (hesp_eval_descs: H2D descriptors, kernels, D2H outcomes + best).
  --impl reference : the unmodified reference (oracle/_ref) on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "simulated schedules/sec (Cholesky DAG) at 1/2/4/8 B200 vs host-CPU ref"
UNIT = "schedules/s"
HARNESS = os.path.join(ROOT, "oracle", "_ref", "ref_harness")
WORKLOAD_DESC = ("C2: random recursive partitionings (K~U[0,8] partition ops, s in {2,4}, depth<=3) "
                 "of the 16x16-tile Cholesky (n=16384, SP) on the CPU-GPU platform model "
                 "(25 cpu + 3 gpu, 4 spaces), PL/EFT-P/WB")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C2")
    ap.add_argument("--batch", type=int, default=100_000, help="candidates per GPU per step")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="CPU baseline sample bound")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        return d.get("hbm_gbs", 6650.0), "measured", d
    return 6650.0, "fallback", {}


def config_block(name, p, n_gpus, batch):
    return {"workload": WORKLOAD_DESC if name == "C2" else name, "preset": name, "n": p["n"],
            "elem_size": p["elem"], "s_base": p["s_base"], "k_max": p["k_max"], "max_depth": p["max_depth"],
            "s_choices": list(p["s_choices"]),
            "policy": f"{p['ordering']}/{p['selection']}/{p['caching']}",
            "platform": p["platform"], "model": p["model"], "batch_per_gpu": batch,
            "global_batch": batch * n_gpus, "parallelism": f"dp{n_gpus} (candidate shards, NCCL min-reduce)",
            "l2": "flushed between steps (256 MiB write), flush outside the timed events"}


def cpu_baseline(p, seconds, first=0):
    """The unmodified reference on this host's cores (oracle/_ref/ref_harness)."""
    from paper_1602_05510_b200.configs import harness_args
    from paper_1602_05510_b200.engine import FIXTURES
    if not os.path.exists(HARNESS):
        return None, "oracle/_ref/ref_harness not built"
    threads = os.cpu_count() or 1
    cmd = [HARNESS, *harness_args(p, FIXTURES), "--first", str(first), "--count", "10000000",
           "--threads", str(threads), "--time-limit", str(seconds)]
    r = subprocess.run(cmd, capture_output=True, text=True, check=True)
    d = json.loads(r.stdout.strip().splitlines()[-1])
    return d, None


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device, self.proc, self.path = device, None, f"/tmp/hesp_clocks_{os.getpid()}.csv"

    def start(self):
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-i", str(self.device), "-lms", "200"], stdout=self.f,
                                         stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None

    def stop(self):
        if not self.proc:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.f.close()
        rows = []
        with open(self.path) as f:
            for line in f:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 9 and parts[1].replace(".", "").isdigit():
                    rows.append(parts)
        if not rows:
            return None
        sm = [float(r[1]) for r in rows]
        mx = max(float(r[2]) for r in rows)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": reasons, "samples": len(rows)}


def algorithmic_bytes(best_steps, P, S, n_types):
    """Scheduler-state bytes per launch:
    B_smem = 8 * sum_t (P + S*k_t + n_types + 4) + 12 * E, summed over the
    candidates of one step from the engine's own counts (leaves, k_t, edges)."""
    leaves = sum(b.sum_leaves for b in best_steps)
    ksum = sum(b.sum_k for b in best_steps)
    edges = sum(b.sum_edges for b in best_steps)
    return (8 * (leaves * (P + n_types + 4) + S * ksum) + 12 * edges) / len(best_steps)


def roofline(best_steps, kernel_ms, P, S, n_types, sm_count, clk, traffic):
    """§8(d)'s binding roofline: the event loop's scheduler-state accesses
    against the chip's shared-memory bandwidth, 128 B/clk per SM at the SM
    clock sampled during the timed region (the kernel is neither HBM- nor
    tensor-bound: compulsory HBM traffic is a descriptor in, 32 B out)."""
    per_launch = algorithmic_bytes(best_steps, P, S, n_types)
    ms = statistics.mean(kernel_ms)
    achieved = per_launch / (ms * 1e-3) / 1e9
    mhz = (clk or {}).get("sm_mhz") or 1965.0
    peak = sm_count * 128 * mhz * 1e6 / 1e9
    return {"bound": "smem", "achieved": round(achieved, 3), "peak": round(peak, 1), "unit": "GB/s",
            "frac": round(achieved / peak, 6), "traffic": traffic,
            "peak_source": f"{sm_count} SMs x 128 B/clk x {mhz:.0f} MHz (sampled SM clock, SURVEY.md §8d)",
            "algorithmic_bytes_per_launch": int(per_launch),
            "kernel": "sim_kernel (event loop; summed over the step's chunks)",
            "kernel_ms_per_launch": round(ms, 4)}


def hbm_roofline(best_steps, kernel_ms, P, S, n_types, peak_gbs, peak_kind, traffic):
    """The same bytes against the measured HBM copy bandwidth (the contract's
    default denominator), with the ncu DRAM traffic of the same kernel."""
    per_launch = algorithmic_bytes(best_steps, P, S, n_types)
    ms = statistics.mean(kernel_ms)
    achieved = per_launch / (ms * 1e-3) / 1e9
    return {"bound": "hbm", "achieved": round(achieved, 3), "peak": peak_gbs, "unit": "GB/s",
            "frac": round(achieved / peak_gbs, 6), "traffic": traffic, "peak_source": peak_kind}


def verify_winner(eng, p, index, makespan):
    """Re-run the reported winner through the unmodified reference
    (oracle/_ref/ref_harness, outside the timed region) and through the
    engine's host-buffer path; the two 40-byte records must be identical."""
    import tempfile
    import numpy as np
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from golden_io import read_golden
    from paper_1602_05510_b200.configs import harness_args
    from paper_1602_05510_b200.engine import FIXTURES
    if index < 0:
        return {"winner_verified": False, "why": "no valid candidate"}
    if not os.path.exists(HARNESS):
        return {"winner_verified": False, "why": "oracle/_ref/ref_harness not built"}
    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, "w.bin")
        subprocess.run([HARNESS, *harness_args(p, FIXTURES), "--first", str(index), "--count", "1",
                        "--threads", "1", "--out", path], check=True, capture_output=True)
        ref = read_golden(path)[0]
    out, _ = eng.eval_descs(eng.generate_host(index, 1), first=index)
    o = out[0]
    same = (int(o["status"]) == int(ref["status"]) == 0 and int(o["n_leaves"]) == int(ref["n_leaves"])
            and np.float64(o["makespan"]).view("<u8") == np.float64(ref["makespan"]).view("<u8")
            and np.float64(makespan).view("<u8") == np.float64(ref["makespan"]).view("<u8")
            and int(o["assign_hash"]) == int(ref["assign_hash"]) and int(o["xfer_hash"]) == int(ref["xfer_hash"]))
    return {"winner_verified": bool(same), "reference_makespan": float(ref["makespan"]),
            "reference_assign_hash": f"{int(ref['assign_hash']):016x}", "reference_xfer_hash": f"{int(ref['xfer_hash']):016x}"}


def issue_roofline(config, value, sm_count, clk):
    """Issue-slot view of the same step (the binding resource):
    warp-instructions per candidate measured by ncu on this config
    (profiles/ncu_issue.json, smsp__inst_executed.sum of build_kernel +
    sim_kernel / candidates) x candidates/s, against SMs x 4 schedulers x the
    SM clock sampled during the timed region."""
    path = os.path.join(ROOT, "profiles", "ncu_issue.json")
    if not os.path.exists(path) or not clk:
        return None
    with open(path) as f:
        d = json.load(f)
    if d.get("config") != config:
        return None
    ipc = d["warp_inst_per_candidate"]
    per_cand = sum(ipc.values())
    peak = sm_count * 4 * clk["sm_mhz"] * 1e6
    ach = per_cand * value
    return {"bound": "issue", "achieved": ach, "peak": peak, "unit": "warp-inst/s", "frac": round(ach / peak, 4),
            "warp_inst_per_candidate": ipc, "source": "profiles/ncu_issue.json (" + d.get("source", "ncu") + ")"}


def ncu_smem(config):
    """Shared-memory and issue counters of the sim kernel from the committed
    ncu capture of this config (profiles/ncu_smem.json), if any."""
    path = os.path.join(ROOT, "profiles", "ncu_smem.json")
    if not os.path.exists(path):
        return None
    with open(path) as f:
        d = json.load(f)
    return d if d.get("config") == config else None


def ncu_traffic(config, batch):
    path = os.path.join(ROOT, "profiles", "ncu_eval_kernel.json")
    if not os.path.exists(path):
        return None
    with open(path) as f:
        d = json.load(f)
    if d.get("config") == config and d.get("batch") == batch:
        return d.get("dram_bytes_per_launch")
    return None


def run_reference(args, p):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    total, wall = 0, 0.0
    per_step = []
    for step in range(args.warmup + args.steps):
        budget = 2.0 if step < args.warmup else args.cpu_seconds
        d, err = cpu_baseline(p, budget, first=step * 1_000_000)
        if err:
            print(json.dumps({"impl": "reference", "unavailable": err}))
            return 0
        if step >= args.warmup:
            total += d["candidates"]
            wall += d["wall_s"]
            per_step.append(d)
    value = total / wall
    threads = per_step[0]["threads"]
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * wall / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": config_block(args.config, p, 1, int(total / args.steps)),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                             "sample": f"{total} candidates of {args.config} over {args.steps} steps of "
                                       f"~{args.cpu_seconds:.0f} s each (time-bounded), {cpu_model()}"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


def main():
    args = parse()
    from paper_1602_05510_b200.configs import CONFIGS
    p = CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference(args, p)

    import numpy as np
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    from paper_1602_05510_b200.dist import init_nccl
    init_nccl(local)  # also at N=1: the winner always goes through hesp_min_reduce over NCCL

    from paper_1602_05510_b200.build import build
    from paper_1602_05510_b200.configs import make_engine
    from paper_1602_05510_b200.engine import DESC_DTYPE, OUTCOME_DTYPE
    if rank == 0:
        build()
    if world > 1:
        dist.barrier()
    eng = make_engine(p, device=local)
    info = eng.info()
    B = args.batch
    nsteps = args.warmup + args.steps
    stream = torch.cuda.Stream()
    # candidate indices: disjoint per (step, rank)
    firsts = [(s * world + rank) * B for s in range(nsteps)]
    descs = torch.empty((nsteps, B * DESC_DTYPE.itemsize), dtype=torch.uint8, device="cuda")
    outs = torch.empty((B * OUTCOME_DTYPE.itemsize,), dtype=torch.uint8, device="cuda")
    with torch.cuda.stream(stream):
        for s in range(nsteps):
            eng.generate_device(firsts[s], B, descs[s].data_ptr(), stream.cuda_stream)
    stream.synchronize()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    from paper_1602_05510_b200.dist import engine_global_best

    def global_best(b):  # K3: hesp_min_reduce over the process group's NCCL communicator
        return engine_global_best(eng, b)[0]

    for s in range(args.warmup):
        b = eng.eval_descs_device(descs[s].data_ptr(), B, firsts[s], outs.data_ptr(), stream.cuda_stream)
        global_best(b)
    launches0 = eng.info().kernel_launches
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    step_ms, kernel_ms, build_ms, bests, winners = [], [], [], [], []
    for s in range(args.warmup, nsteps):
        with torch.cuda.stream(stream):
            flush.fill_(s & 0xff)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        b = eng.eval_descs_device(descs[s].data_ptr(), B, firsts[s], outs.data_ptr(), stream.cuda_stream)
        winners.append(global_best(b))
        e1.record(stream)
        e1.synchronize()
        step_ms.append(e0.elapsed_time(e1))
        kernel_ms.append(b.sim_ms if b.sim_ms > 0 else b.kernel_ms)
        build_ms.append(b.build_ms)
        bests.append(b)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    launches = eng.info().kernel_launches - launches0
    total_ms = sum(step_ms)
    t = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    max_ms = float(t.item())
    value = world * B * args.steps / (max_ms * 1e-3)

    # ---- e2e through the C ABI with host buffers (H2D descs, D2H outcomes) ----
    host_descs = [eng.generate_host(firsts[s], B) for s in range(args.warmup, nsteps)]
    for w in range(max(1, args.warmup)):  # warm the host path (pinned staging, page tables) like the device path
        eng.eval_descs(host_descs[w % len(host_descs)], first=firsts[args.warmup + w % len(host_descs)])
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e2e_steps = []
    t0 = time.perf_counter()
    for i, s in enumerate(range(args.warmup, nsteps)):
        ts = time.perf_counter()
        out, b = eng.eval_descs(host_descs[i], first=firsts[s])
        global_best(b)
        e2e_steps.append(round(1e3 * (time.perf_counter() - ts), 2))
    e2e_s = time.perf_counter() - t0
    # descriptors travel packed (offsets + used ops); count what was copied
    h2d_bytes = int(eng.info().last_h2d_bytes)
    te = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = world * B * args.steps / float(te.item())

    if rank == 0:
        peak, peak_kind, _ = measured_peaks()
        P = eng._pc.n_procs
        traffic = ncu_traffic(args.config, B)
        rf = roofline(bests, kernel_ms, P, eng._pc.n_spaces, eng._pc.n_types, info.sm_count, clk, traffic)
        rf["build_kernel_ms_per_step"] = round(statistics.mean(build_ms), 4) if build_ms else None
        rf["ncu"] = ncu_smem(args.config)
        hrf = hbm_roofline(bests, kernel_ms, P, eng._pc.n_spaces, eng._pc.n_types, peak, peak_kind, traffic)
        winner = verify_winner(eng, p, winners[-1][1], winners[-1][0])
        cpu = None
        if not args.no_cpu_baseline and world == 1:  # rank 0 at N=1 only
            d, err = cpu_baseline(p, args.cpu_seconds)
            if d:
                cpu = {"value": d["cand_per_s"], "unit": UNIT, "cores": d["threads"], "kind": "reference",
                       "sample": f"{d['candidates']} candidates of {args.config} (indices 0..), "
                                 f"time-bounded {args.cpu_seconds:.0f} s, {d['threads']} threads, {cpu_model()}"}
            else:
                cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference", "sample": err}
        n_ok = sum(b.n_ok for b in bests)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": max_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_block(args.config, p, world, B),
            "e2e": {"value": e2e_value, "unit": UNIT,
                    "h2d_bytes_per_step": h2d_bytes,
                    "d2h_bytes_per_step": B * OUTCOME_DTYPE.itemsize + 64, "step_ms": e2e_steps},
            "gpu_launches": int(launches),
            "roofline": rf,
            "hbm_roofline": hrf,
            "issue_roofline": issue_roofline(args.config, value, info.sm_count, clk),
            "cpu_baseline": cpu,
            "clocks": clk,
            "valid_fraction": n_ok / (B * args.steps),
            "valid_per_s": value * n_ok / (B * args.steps),
            "counting": "value counts every evaluated candidate (as the reference arm does); valid_per_s only "
                        "those the reference simulates without an Err (the rest end in CoherenceError)",
            "best": {"makespan": winners[-1][0], "index": winners[-1][1], **winner},
            "min_reduce": {"backend": "nccl", "world": world, "calls": int(eng.info().min_reduces)},
            "engine": {"slots": info.n_slots, "sm_count": info.sm_count, "blocks_per_sm": info.blocks_per_sm,
                       "warps_per_block": info.warps_per_block, "slot_bytes": info.slot_bytes,
                       "chunk": info.chunk, "kernels": "build_kernel + sim_kernel per chunk" if info.chunk else "eval_kernel"},
        }
        print(json.dumps(line))
    dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
