#!/usr/bin/env python3
"""Benchmark of the rehearsal-buffer hot path (update + unbiased global sample + augmented
batch), BASELINE.json metric "augmented samples/sec (update+global sample)".

Our arm (default): one process per GPU (torchrun for N>1). A step is one engine iteration
on every rank: insert candidates of m_i, publish occupancy, draw reps(i-1) from the global
buffer, materialise m'_i = m_i ++ reps(i-1) (one fused sm_100a launch per rank, issued from
native code over a device-resident input ring larger than L2). value = augmented samples
produced by all ranks / max-over-ranks device time. e2e = the same through the host-buffer
C-ABI call (drb_rb_step_host: pinned host m_i in, m'_i back to pinned host memory).

Reference arm (--impl reference): the unmodified reference C++ engine (oracle/_ref,
compiled from /root/reference sources) — N in-process workers over loopback TCP, each
doing engine.update(m) + augment(m, reps) — on rank 0's host cores, bounded sample.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# BASELINE.json configs[1] (the metric's named config), parameters per SURVEY.md §8d:
# ImageNet-100 shape 224x224x3 uint8, K=100 in 4 class-incremental tasks, b=56, r=7, c=14,
# |B| = 30% of ImageNet-100 (~130k) spread over 8 GPUs -> 4875 per GPU -> cap 48 per class.
CONFIGS = {
    "c2": dict(workload="imagenet100-224x224x3-u8-class-incremental", K=100, T=4, cap=48, S=224 * 224 * 3,
               dtype="u8", b=56, r=7, c=14),
    "c1": dict(workload="synthetic-32x32x3-fp32", K=10, T=1, cap=100, S=32 * 32 * 3 * 4, dtype="f32",
               b=64, r=8, c=14),
    "c3": dict(workload="imagenet1k-224x224x3-u8-10pct-per-gpu", K=1000, T=4, cap=128, S=224 * 224 * 3,
               dtype="u8", b=56, r=7, c=14),
    "c4": dict(workload="imagenet100-224x224x3-fp16-b128-r28", K=100, T=4, cap=48, S=224 * 224 * 3 * 2,
               dtype="f16", b=128, r=28, c=14),
    "c4r14": dict(workload="imagenet100-224x224x3-fp16-b128-r14", K=100, T=4, cap=48, S=224 * 224 * 3 * 2,
                  dtype="f16", b=128, r=14, c=14),
    "c4r7": dict(workload="imagenet100-224x224x3-fp16-b128-r7", K=100, T=4, cap=48, S=224 * 224 * 3 * 2,
                 dtype="f16", b=128, r=7, c=14),
    "c5": dict(workload="sensor-128x128x1-fp32", K=50, T=1, cap=40, S=128 * 128 * 4, dtype="f32",
               b=256, r=32, c=14),
}
METRIC = "augmented samples/sec (update+global sample)"
UNIT = "aug_samples/s"


def hbm_bytes_per_step(cfg) -> int:
    """SURVEY.md §8d algorithmic HBM bytes per rank per iteration: 2*S*(c + r + b)."""
    return 2 * cfg["S"] * (cfg["c"] + cfg["r"] + cfg["b"])


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_dev{device}_{os.getpid()}.csv")

    def __enter__(self):
        if os.environ.get("BENCH_NO_CLOCKS"):  # (experiments: the timed region without the sampler)
            return self
        os.makedirs(os.path.dirname(self.path), exist_ok=True)
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
            time.sleep(0.3)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.1)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.f.close()

    def summary(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        rows = []
        with open(self.path) as f:
            for line in f:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) == 6 and parts[0].isdigit():
                    rows.append(parts)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = sorted(int(r[0]) for r in rows)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": int(rows[0][1]), "reasons": reasons, "samples": len(rows)}


class NvlinkCounters:
    """NVLink data bytes sent / received by one GPU (NVML field values, summed over its links):
    the hardware's count of what the pushes put on the wire, read around the timed region."""

    def __init__(self, device: int, links: int = 18):
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.fields = [(f, l) for f in (pynvml.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX,
                                            pynvml.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX) for l in range(links)]
            self.read()
            self.ok = True
        except Exception as e:  # noqa: BLE001
            self.err = f"{type(e).__name__}: {e}"

    def read(self):
        vals = self.nv.nvmlDeviceGetFieldValues(self.h, self.fields)
        tx = rx = 0
        bad = [int(v.nvmlReturn) for v in vals if v.nvmlReturn != 0]
        if len(bad) == len(vals):
            raise RuntimeError(f"NVML field values unsupported (return {bad[0]})")
        for k, v in enumerate(vals):
            if v.nvmlReturn != 0:
                continue
            x = int(v.value.ullVal) * 1024  # KiB
            if k < len(self.fields) // 2:
                tx += x
            else:
                rx += x
        return tx, rx


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return world, rank, local


def load_workload():
    """paper_2406_03285_b200/workload.py (numpy input generation) loaded by path, so the
    reference arm never runs the package __init__ (which maps libdrb_b200.so)."""
    import importlib.util
    path = os.path.join(ROOT, "paper_2406_03285_b200", "workload.py")
    spec = importlib.util.spec_from_file_location("drb_bench_workload", path)
    mod = importlib.util.module_from_spec(spec)
    sys.modules["drb_bench_workload"] = mod
    spec.loader.exec_module(mod)
    return mod


STEPS_PER_TASK = 100


def bench_config(cfg, n_gpus: int, ring: int):
    """The one `config` both arms print (same workload, same keys)."""
    K, cap, S, b = cfg["K"], cfg["cap"], cfg["S"], cfg["b"]
    return {"workload": cfg["workload"], "K": K, "cap": cap, "b": b, "r": cfg["r"], "c": cfg["c"], "S": S,
            "tasks": cfg["T"], "steps_per_task": STEPS_PER_TASK,
            "prefill_steps": cfg["T"] * STEPS_PER_TASK,
            "parallelism": f"dp{n_gpus}" if n_gpus > 1 else "single",
            "l2": f"inputs larger than L2: {ring}-batch device ring ({ring * b * S / 2**20:.0f} MiB), "
                  f"slab {K * cap * S / 2**20:.0f} MiB per GPU"}


def host_info():
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        avail = len(os.sched_getaffinity(0))
    except AttributeError:
        avail = os.cpu_count() or 1
    return {"cpu_model": model, "nproc": avail, "cpu_count": os.cpu_count()}


def cpu_baseline_sample(cfg, n_workers: int, iters: int):
    """Reference engine on the host cores (oracle/_ref): N in-process workers over loopback
    TCP, each doing engine.update(m) + augment(m, reps) (proj/tests/test_engine.cpp:57-107,
    proj/src/runner/overlap.cpp:83-89 with zero train cost), after a prefill of
    T x steps_per_task steps whose labels cycle through every task, so every class is at
    capacity (replacements) as in the GPU arm. Falls back to the C port's replay."""
    from oracle.py_oracle import Backend, have_reference
    wl = load_workload()
    spec = wl.stream_spec(cfg["K"], cfg["T"], cfg["b"], cfg["S"], steps_per_task=STEPS_PER_TASK, seed=1)
    ring = 8
    prefill = cfg["T"] * STEPS_PER_TASK

    def step_of(i):  # ring slot i covers task i % T
        return (i % cfg["T"]) * STEPS_PER_TASK + i
    data = np.stack([np.stack([spec.payload(w, step_of(i)) for i in range(ring)]) for w in range(n_workers)])
    labels = np.stack([np.stack([spec.labels(w, step_of(i)) for i in range(ring)]) for w in range(n_workers)])
    info = host_info()
    if have_reference():
        be = Backend("reference")
        secs, samples = be.engine_bench(n_workers, cfg["K"], cfg["cap"], cfg["S"], cfg["b"], cfg["c"], cfg["r"],
                                        1, data, labels, prefill, iters)
        # per worker: the training thread and the engine's pipeline thread are the busy ones
        kind, cores = "reference", min(2 * n_workers, info["nproc"])
    else:
        be = Backend("port")
        rp = be.replay(n_workers, cfg["K"], cfg["cap"], cfg["S"], cfg["c"], cfg["r"], 1)
        for i in range(prefill):
            rp.step(data[:, i % ring], labels[:, i % ring])
        t0 = time.perf_counter()
        samples = 0
        for i in range(iters):
            _, _, cnt = rp.step(data[:, i % ring], labels[:, i % ring])
            samples += int(cnt.sum())
        secs = time.perf_counter() - t0
        kind, cores = "port", 1
    return {"value": samples / secs, "unit": UNIT, "cores": cores, "kind": kind, **info,
            "n_workers": n_workers, "seconds": secs,
            "sample": f"{iters} timed iterations x {n_workers} in-process worker(s) of {cfg['workload']} after a "
                      f"{prefill}-step prefill to capacity (f32-packed payload, same byte volume), {samples} "
                      f"augmented samples in {secs:.2f}s"}


def run_reference(args, cfg):
    world, rank, _ = dist_env()
    n = args.gpus if args.gpus else world
    if rank != 0:
        return 0
    try:
        iters = max(1, min(args.steps, args.ref_iters))
        cb = cpu_baseline_sample(cfg, n, iters)
    except Exception as e:  # noqa: BLE001
        emit({"impl": "reference", "unavailable": f"{type(e).__name__}: {e}"})
        return 0
    step_samples = (cfg["b"] + cfg["r"]) * n  # steady state: every worker's m' has b + r rows
    line = {"impl": "reference", "metric": METRIC, "value": cb["value"], "unit": UNIT, "n_gpus": n,
            "steps": iters, "warmup": cfg["T"] * STEPS_PER_TASK,
            "ms_per_step": 1000.0 * step_samples / cb["value"] if cb["value"] else None,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": cfg["dtype"],
            "data": "synthetic", "config": bench_config(cfg, n, args.ring),
            "cpu_baseline": cb, "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                                        "d2h_bytes_per_step": 0},
            "gpu_launches": 0}
    emit(line)
    return 0


_JSON_FD = 1


def emit(line):
    """The one JSON line, on the process's original stdout (library chatter such as NCCL's version
    banner is routed to stderr by quiet_stdout)."""
    os.write(_JSON_FD, (json.dumps(line) + "\n").encode())


def quiet_stdout():
    global _JSON_FD
    sys.stdout.flush()
    _JSON_FD = os.dup(1)
    os.dup2(2, 1)


def main():
    quiet_stdout()
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=0)
    ap.add_argument("--steps", type=int, default=20000)
    ap.add_argument("--warmup", type=int, default=50)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--ring", type=int, default=64, help="device input batches (>L2 in total)")
    ap.add_argument("--e2e-steps", type=int, default=500)
    ap.add_argument("--cpu-iters", type=int, default=200)
    ap.add_argument("--sweep", default="", help="comma-separated step counts: also time one run of each "
                                                "(fixed per-run cost vs steps; reported as steps_sweep)")
    ap.add_argument("--ref-iters", type=int, default=400)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="issue the timed launches one by one")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference(args, cfg)

    import torch
    import torch.distributed as dist

    import paper_2406_03285_b200 as drb
    from paper_2406_03285_b200.workload import stream_spec

    world, rank, local = dist_env()
    N = world
    if args.gpus and args.gpus != world:
        if world == 1 and args.gpus > 1:
            raise SystemExit("bench.py --gpus N>1 must be launched under torchrun (one process per GPU)")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", init_method="env://", device_id=torch.device(f"cuda:{local}"))

    K, cap, S, b, r, c = cfg["K"], cfg["cap"], cfg["S"], cfg["b"], cfg["r"], cfg["c"]
    steps_per_task = STEPS_PER_TASK
    spec = stream_spec(K, cfg["T"], b, S, steps_per_task=steps_per_task, seed=1)
    # the whole GPU for the engine: the bench has no training step to share the SMs with
    engine_ctas = torch.cuda.get_device_properties(local).multi_processor_count
    # the default 32 m' slots: in the split update() form the loader may run 30 steps ahead of
    # the trainer (16 slots: 6.2 instead of 5.9 us per pipelined update; runs are unaffected)
    aug_ring = 32
    buf = drb.rehearsal_buffer(K, cap, S, max_batch=b, candidate_count=c, rep_count=r, seed=1, rank=rank,
                               world=N, device=local, engine_ctas=engine_ctas, aug_ring=aug_ring)
    if N > 1:
        from paper_2406_03285_b200.dist import connect_world
        connect_world(buf)
    eng = drb.engine(buf)
    eng.start()

    ring = args.ring
    from paper_2406_03285_b200.workload import device_ring
    data, _ = device_ring(spec, rank, ring, f"cuda:{local}")
    # Labels follow the class-incremental schedule. The ring of labels is re-drawn per
    # phase so prefill visits every task (buffers fill) and the timed region sits in one.
    def labels_for(first):
        return torch.from_numpy(np.stack([spec.labels(rank, first + i) for i in range(ring)]).astype(np.int32)).cuda(local)

    stream = torch.cuda.Stream(device=local)
    torch.cuda.synchronize()

    def barrier():
        if N > 1:
            dist.barrier(device_ids=[local])

    # prefill: every task's classes fill to capacity (replacements dominate afterwards)
    step = 0
    prefill = cfg["T"] * steps_per_task
    while step < prefill:
        lab = labels_for(step)
        cnt = min(ring, prefill - step)
        eng.run(data[:cnt], lab[:cnt], cnt, first=0, stream=stream)
        step += cnt
        stream.synchronize()
    lab = labels_for(step)
    # The clock sampler starts before the warm-up steps (it needs ~0.3 s to produce samples): the
    # GPUs then go from the warm-up straight into the timed region instead of idling while it
    # starts, which would time the first microseconds of the region at ramping clocks.
    nvl = NvlinkCounters(local)  # (NVML init here, not between the warm-up and the timed region)
    clocks = ClockSampler(local)
    late_clocks = bool(os.environ.get("BENCH_CLOCKS_LATE"))  # (experiments: the old order)
    if not late_clocks:
        clocks.__enter__()
    eng.run(data, lab, args.warmup, first=0, stream=stream)
    step += args.warmup
    stream.synchronize()
    barrier()

    # timed region: K steps, back to back, device-timed (events on the launching stream).
    # The K launches are captured into a CUDA graph beforehand (host launch cost paid
    # outside the timed region, as a training loop would replay a captured step).
    resident = eng.engine_info()["resident"]
    run = eng.prepare_run(data, lab, args.steps, first=args.warmup) if not args.no_graph else None
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    if late_clocks:
        clocks.__enter__()
    try:
        # NVML counters before the barrier: a slow NVML query must not skew the ranks' starts
        nvl0 = nvl.read() if (nvl.ok and N > 1) else None
        barrier()
        torch.cuda.synchronize()
        inst0 = eng.engine_info()["instances"]
        ev0.record(stream)
        if run is not None:
            run.launch(stream)
        else:
            eng.run(data, lab, args.steps, first=args.warmup, stream=stream)
        ev1.record(stream)
        torch.cuda.synchronize()
        barrier()
    finally:
        clocks.__exit__(None, None, None)
    timed_instances = eng.engine_info()["instances"] - inst0
    nvl1 = nvl.read() if (nvl.ok and N > 1) else None
    if run is not None:
        run.close()
    t_ms = ev0.elapsed_time(ev1)
    step += args.steps
    if N > 1:
        tt = torch.tensor([t_ms], device=f"cuda:{local}", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_ms = float(tt.item())
    nvlink = None
    if N > 1:
        if nvl.ok:
            tt = torch.tensor([nvl1[0] - nvl0[0], nvl1[1] - nvl0[1]], device=f"cuda:{local}", dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.SUM)
            # algorithmic: every rank receives r*S*(N-1)/N per step (the reps its peers own)
            nvlink = {"tx_bytes_per_step_per_rank": float(tt[0]) / N / args.steps,
                      "rx_bytes_per_step_per_rank": float(tt[1]) / N / args.steps,
                      "algorithmic_bytes_per_step_per_rank": r * S * (N - 1) / N,
                      "rx_gbs_per_rank": float(tt[1]) / N / (t_ms / 1000.0) / 1e9 if t_ms else None,
                      "peak_gbs_per_direction": 900.0,
                      "source": "NVML NVLink data throughput counters, summed over links, around the timed region"}
        else:
            nvlink = {"unavailable": nvl.err}
    samples = (b + r) * N * args.steps  # steady state: every rank's m'_i has b + r rows
    value = samples / (t_ms / 1000.0)
    ms_per_step = t_ms / args.steps

    # fixed per-run cost: the same timed region (sync + barrier, one prepared run, events on
    # its stream) for several run lengths; us_per_step(K) = t(K) / K
    sweep = []
    for ks in [int(x) for x in args.sweep.split(",") if x.strip()]:
        sr = eng.prepare_run(data, lab, ks, first=0) if not args.no_graph else None
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        c0 = nvl.read() if (nvl.ok and N > 1) else None  # (before the barrier: no rank skew)
        barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        if sr is not None:
            sr.launch(stream)
        else:
            eng.run(data, lab, ks, first=0, stream=stream)
        e1.record(stream)
        torch.cuda.synchronize()
        c1 = nvl.read() if (nvl.ok and N > 1) else None
        if sr is not None:
            sr.close()
        tk = e0.elapsed_time(e1)
        ent = {"steps": ks}
        if N > 1:
            tt = torch.tensor([tk], device=f"cuda:{local}", dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            tk = float(tt.item())
            if c0 is not None:
                cc = torch.tensor([c1[0] - c0[0], c1[1] - c0[1]], device=f"cuda:{local}", dtype=torch.float64)
                dist.all_reduce(cc, op=dist.ReduceOp.SUM)
                ent["nvlink_rx_bytes_per_step_per_rank"] = float(cc[1]) / N / ks
                ent["nvlink_tx_bytes_per_step_per_rank"] = float(cc[0]) / N / ks
        step += ks
        ent.update({"ms": tk, "us_per_step": 1000.0 * tk / ks})
        sweep.append(ent)

    # The drop-in API a trainer calls (trainer.cpp:109-113): update(m_i) on one stream, one call
    # per step, serial (the next post follows the previous m' on the stream, as in a training
    # loop with zero train cost), inputs resident in HBM, device-timed like the run above.
    # Also split: the loader's stream posts m_i, the trainer's stream (here: with no training)
    # releases the m' it used and waits for m'_i (drb_rb_step_split), so posts pipeline.
    producer = torch.cuda.Stream(device=local)

    def time_updates(nsteps, split=False):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        torch.cuda.synchronize()
        inst0 = eng.engine_info()["instances"]
        e0.record(stream)
        if split:
            producer.wait_stream(stream)  # the timed region starts at e0 for the producer too
        for k in range(nsteps):
            if split:
                eng.update((data[k % ring], lab[k % ring]), stream=producer, consumer=stream)
            else:
                eng.update((data[k % ring], lab[k % ring]), stream=stream)
        e1.record(stream)
        torch.cuda.synchronize()
        tk = e0.elapsed_time(e1)
        if N > 1:
            tt = torch.tensor([tk], device=f"cuda:{local}", dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            tk = float(tt.item())
        return 1000.0 * tk / nsteps, eng.engine_info()["instances"] - inst0
    # the same through the C++ facade (tools/update_bench: the reference's trainer is C++; no
    # Python in the per-step path), N=1 only: 2000 steps (the steady state of a training loop;
    # it also reports 20 steps)
    cpp_update = None
    exe = os.path.join(ROOT, "tools", "update_bench")
    if N == 1 and os.path.exists(exe) and not os.environ.get("BENCH_NO_CPP"):
        try:
            res = subprocess.run([exe, "2000", str(local), str(aug_ring)], capture_output=True, text=True,
                                 timeout=300)
            cpp_update = json.loads(res.stdout.strip().splitlines()[-1]) if res.returncode == 0 else \
                {"error": res.stderr[-300:]}
        except Exception as e:  # noqa: BLE001
            cpp_update = {"error": f"{type(e).__name__}: {e}"}
    upd_serial_us, upd_launch = time_updates(args.steps)
    upd_serial_us_200, _ = time_updates(200)
    upd_us, upd_split_launch = time_updates(args.steps, split=True)
    upd_us_200, _ = time_updates(200, split=True)
    step += 2 * (args.steps + 200)
    kernel_ms = None
    if not resident:  # three-kernel path: per-launch copy-kernel times from events in the graph
        nper = 256
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(2 * nper)]
        for e in evs:  # torch creates the CUDA event lazily on first record
            e.record(stream)
        stream.synchronize()
        barrier()
        krun = eng.prepare_run(data, lab, nper, first=0, events=evs)
        krun.launch(stream)
        torch.cuda.synchronize()
        krun.close()
        launch_ms = [evs[2 * i].elapsed_time(evs[2 * i + 1]) for i in range(nper)]
        kernel_ms = float(np.median(launch_ms))
        step += nper
        if N > 1:
            tt = torch.tensor([kernel_ms], device=f"cuda:{local}", dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            kernel_ms = float(tt.item())

    # e2e through the host-buffer C-ABI call drb_rb_step_host: pinned host m_i in, m'_i
    # assembled in place in the caller's buffer (rows [0, b) are m_i, the r representative
    # rows and their labels come back over PCIe) — reps = update(m); m' = augment(m, reps)
    e2e_steps = args.e2e_steps
    hring = 4
    h_slot = torch.empty((hring, b + r, S), dtype=torch.uint8).pin_memory()
    h_slot[:, :b].copy_(data[:hring].cpu())
    h_lab = torch.empty((hring, b + r), dtype=torch.int32).pin_memory()
    h_lab[:, :b].copy_(lab[:hring].cpu())
    h_cnt = torch.zeros(hring, dtype=torch.int32).pin_memory()
    hs, hl, hc = (x.numpy() for x in (h_slot, h_lab, h_cnt))

    def host_step(i):
        k = i % hring
        eng.update_host(hs[k][:b], hl[k][:b].view(np.uint32), hs[k], hl[k].view(np.uint32),
                        hc[k:k + 1].view(np.uint32))
    for i in range(8):  # warm
        host_step(i)
    eng.synchronize()
    barrier()
    t0 = time.perf_counter()
    for i in range(e2e_steps):
        host_step(i)
    eng.synchronize()
    e2e_s = time.perf_counter() - t0
    if N > 1:
        tt = torch.tensor([e2e_s], device=f"cuda:{local}", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_s = float(tt.item())
    e2e_value = (b + r) * N * e2e_steps / e2e_s
    eng.shutdown()

    # PCIe ceiling of the e2e leg: the same H2D + D2H bytes as one step, plain pinned copies
    h2d_b, d2h_b = b * (S + 4), r * (S + 4) + 4
    pin_in = torch.empty(h2d_b, dtype=torch.uint8).pin_memory()
    pin_out = torch.empty(d2h_b, dtype=torch.uint8).pin_memory()
    dev_in = torch.empty(h2d_b, dtype=torch.uint8, device=f"cuda:{local}")
    dev_out = torch.empty(d2h_b, dtype=torch.uint8, device=f"cuda:{local}")
    s_in, s_out = torch.cuda.Stream(device=local), torch.cuda.Stream(device=local)
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            with torch.cuda.stream(s_in):
                dev_in.copy_(pin_in, non_blocking=True)
            with torch.cuda.stream(s_out):
                pin_out.copy_(dev_out, non_blocking=True)
        torch.cuda.synchronize()
        pcie_s = time.perf_counter() - t0
    pcie_steps_per_s = e2e_steps / pcie_s
    # our kernels inside the timed region: the resident engine's instances launched there (one
    # cooperative kernel per busy period; steps are posted with stream memory operations), or
    # sel + plan + copy per step on the three-kernel path (DRB_PERSIST=0)
    launches = timed_instances if resident else 3 * args.steps
    launch_mode = "resident-cooperative" if resident else ("cuda-graph" if not args.no_graph else "direct")
    peak, peak_kind = peaks()
    bytes_step = hbm_bytes_per_step(cfg)
    # The copy kernel is the only bulk kernel and runs back to back, one launch per step, so
    # its average launch duration over the timed region (CUDA events on its stream around
    # exactly K launches) is ms_per_step; this bounds the kernel-only time from above.
    # (Events recorded between single launches inside the graph add node overhead, so the
    # bracketed per-launch figure is reported separately and not used for the fraction.)
    achieved = bytes_step / (ms_per_step / 1000.0) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", f"ncu_traffic_{args.config}.json")
    if os.path.exists(tpath):
        try:
            tj = json.load(open(tpath))
            # DRAM bytes of the dominant kernel per launch, like `achieved`: the timed launch runs
            # K steps, the capture holds the per-step figure of a 200-step instance
            traffic = tj["dram_bytes_per_step"] * (args.steps if resident else 1) if "dram_bytes_per_step" in tj \
                else tj.get("dram_bytes_per_launch")
        except Exception:
            traffic = None

    cpu = None
    if rank == 0 and N == 1 and not args.no_cpu:
        try:
            cpu = cpu_baseline_sample(cfg, 1, args.cpu_iters)
        except Exception as e:  # noqa: BLE001
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "unavailable", "sample": str(e)}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": N, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": cfg["dtype"], "data": "synthetic",
            "config": bench_config(cfg, N, ring),
            "gpu_launches": launches,
            "engine": eng.engine_info(),
            "launch_mode": launch_mode,
            "update_us_per_step": (cpp_update["split_us_per_step"] if cpp_update and "split_us_per_step" in cpp_update
                                   else upd_us),
            "update": {"cpp_facade": cpp_update,
                       "us_per_step": upd_us, "steps": args.steps, "us_per_step_200": upd_us_200,
                       "instances_launched": upd_split_launch,
                       "api": "engine.update(m_i, stream=loader, consumer=trainer) per step (drb_rb_step_split: "
                              "the descriptor is posted on the loader's stream, the trainer's stream releases "
                              "the m' it used and waits for m'_i; no kernel launch per step), inputs resident "
                              "in HBM, device-timed on the trainer's stream",
                       "serial": {"us_per_step": upd_serial_us, "us_per_step_200": upd_serial_us_200,
                                  "instances_launched": upd_launch,
                                  "api": "engine.update(m_i) on one stream (drb_rb_step): each post follows "
                                         "the wait for the previous m' — the latency of one round"}},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d_b,
                    "d2h_bytes_per_step": d2h_b, "steps": e2e_steps,
                    "api": "drb_rb_step_host, m' assembled in place in the caller's pinned batch buffer",
                    "pcie_ceiling": {"value": (b + r) * N * pcie_steps_per_s, "unit": UNIT,
                                     "h2d_gbs": h2d_b * pcie_steps_per_s / 1e9,
                                     "how": "the same per-step H2D and D2H bytes as plain pinned cudaMemcpyAsync "
                                            "on two streams, no kernels"}},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_kind,
                         "algorithmic_bytes_per_step": bytes_step,
                         "algorithmic_bytes_per_launch": bytes_step * (args.steps if resident else 1),
                         "kernel_ms_per_step": ms_per_step,
                         "kernel": "drb_run_kernel" if resident else "drb_copy_tma_kernel",
                         "timing": ("the resident engine processes the K steps of the timed region (its instance "
                                    "launch, pipeline fill and drain included); CUDA events on the posting stream / K"
                                    if resident else "CUDA events over the timed region / K steps"),
                         **({"three_kernel_copy_ms_event_bracketed": kernel_ms} if kernel_ms is not None else {}),
                         "bytes_formula": "2*S*(b+r+c) per rank per iteration (SURVEY.md 8d)"},
            "cpu_baseline": cpu,
            "clocks": clocks.summary(),
            **({"nvlink": nvlink} if nvlink else {}),
            **({"steps_sweep": sweep} if sweep else {}),
        }
        emit(line)
    if N > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
