"""bench.py — LF-MMI loss+gradient throughput on B200 (BASELINE.json metric).

Metric: forward-backward frames×seqs/sec on the denominator graph, B = 128
utterances per GPU (weak scaling), measured as the whole hot path of SURVEY §8(a):
numerator + denominator forward-backward, posteriors, LF-MMI gradient, loss and
totals (+ NCCL all-reduce of the 5 totals when N > 1).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

Workload (SURVEY §8(d) C4, configs[3]): den K=3000 / nnz=20000 (2% hub skew),
pdf map 3000→2000, 128 numerator graphs (L ~ U[50,150] phones), φ [128,500,2000]
U[-10,0) fp32, all N_b = 500; rank r draws its own batch (seed 4 + 1000 r).
Inputs (φ 512 MB, grad 512 MB, α̂ 768 MB per step) exceed the 126 MB L2.

The reference arm (--impl reference) is the float64 C oracle (oracle/) run on
this host's cores over a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import os
import shutil
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

B, N, D, K_DEN, NNZ_DEN = 128, 500, 2000, 3000, 20000
METRIC = "forward-backward frames×seqs/sec (den graph, B=128) & % HBM roofline @1/2/4/8 GPU"
WORKLOAD = "C4: LF-MMI loss+grad, den K=3000 nnz=20000 (pdf 3000→2000) + 128 numerator graphs, φ[128,500,2000] fp32 per GPU"
WORKLOAD_C3 = ("C3: den-only forward + backward with fused state posteriors (fb_forward + fb_backward), K=3000 "
               "nnz=20000 identity pdf map, φ[128,500,3000] fp32 per GPU")
WORKLOAD_N2 = ("N2 (paper Table 1 shape, P:445-457): LF-MMI loss+grad, den K=3022 nnz=50984 (pdf →84) + 128 numerator "
               "graphs of ≈454 states, φ[128,700,84] fp32 per GPU")


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d.get("hbm_gbs", 6650.0)), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
            t0 = time.time()  # nvidia-smi is up (first row) before the timed region starts
            while not self.rows and time.time() - t0 < 5.0:
                time.sleep(0.01)
            self.rows.clear()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def make_c5_batch(rank: int, world: int, mode: str):
    """C5: 1024 variable-length utterances (N_b clipped log-normal,
    median 250, [50, 700]); strong scaling shards all 1024 over the ranks, weak
    scaling the first 128·world.  LPT sharding by N_b·(nnz_den + nnz_num)."""
    from paper_2112_00709_b200 import dist as fdist
    from paper_2112_00709_b200 import synth

    lens, nums, den = synth.make_c5_utterances(seed=5, B=1024, D=D, K=K_DEN, nnz=NNZ_DEN)
    pool = np.arange(1024) if mode == "c5-strong" else np.arange(min(1024, 128 * world))
    costs = fdist.utterance_costs(lens[pool], [nums[i].nnz for i in pool], den.nnz)
    idx = pool[fdist.lpt_shard(costs, world)[rank]]
    n_max = int(lens[idx].max())
    emis = synth.c5_emissions(5, idx, n_max, D)
    return synth.Workload("C5", len(idx), n_max, D, lens[idx].astype(np.int32), emis, den=den,
                          nums=[nums[i] for i in idx])


def make_batch(rank: int, world: int = 1, mode: str = "c4"):
    from paper_2112_00709_b200 import synth

    if mode == "paper":
        # N2: the paper's Table 1 shape; rank r draws its own numerators / emissions
        w = synth.make_paper_shape(seed=6)
        if rank:
            rng = np.random.Generator(np.random.PCG64(6 + 1000 * rank))
            w.nums = [synth.numerator_graph(rng, int(rng.integers(190, 211)), 84, "random", k_max=454)
                      for _ in range(w.B)]
            w.emis = synth.emissions(rng, w.B, w.N_max, 84)
        return w
    if mode == "c2":
        # C2 (configs[1]): 64 left-to-right numerator graphs (G = B), N_b ~ U[max(120, L), 180], D = 300
        w = synth.make_c2(seed=2)
        if rank:
            w.emis = synth.emissions(np.random.Generator(np.random.PCG64(2 + 1000 * rank)), w.B, w.N_max, w.D)
        w.den = synth.compose(w.nums)  # the graph batch the public fb_forward / fb_backward calls take
        return w
    if mode == "viterbi":
        return make_batch(rank, world, "c3")
    if mode == "viterbi-paper":
        return make_batch(rank, world, "paper")
    if mode == "c3":
        # C3 (configs[2]): shared den K=3000 / nnz=20000, identity pdf map, φ [128,500,3000]
        w = synth.make_c3(seed=3, B=B, N=N, K=K_DEN, nnz=NNZ_DEN)
        if rank:
            w.emis = synth.emissions(np.random.Generator(np.random.PCG64(3 + 1000 * rank)), B, N, w.D)
        return w
    if mode != "c4":
        return make_c5_batch(rank, world, mode)

    w = synth.make_c4(seed=4, B=B, N=N, K=K_DEN, nnz=NNZ_DEN, D=D)
    if rank:
        # rank r: same denominator graph, its own numerator graphs and emissions
        rng = np.random.Generator(np.random.PCG64(4 + 1000 * rank))
        w.nums = [synth.numerator_graph(rng, int(rng.integers(50, 151)), D, "random") for _ in range(B)]
        w.emis = synth.emissions(rng, B, N, D)
    return w


# ---------------------------------------------------------------------------- reference arm

def cpu_oracle_rate(w, n_utts: int, threads: int):
    """Oracle seq-frames/s on the first n_utts utterances of the batch."""
    import oracle
    from paper_2112_00709_b200 import synth

    os.environ["OMP_NUM_THREADS"] = str(threads)
    oracle.lib()
    num = synth.compose(w.nums[:n_utts])
    den = synth.compose([w.den])
    t0 = time.perf_counter()
    r = oracle.lfmmi_batch(num, den, w.emis[:n_utts], w.lengths[:n_utts])
    dt = time.perf_counter() - t0
    assert (r["status"] == 0).all()
    return float(w.lengths[:n_utts].sum()) / dt, dt


def run_reference(args, rank, world):
    if rank != 0:
        return
    threads = len(os.sched_getaffinity(0))
    w = make_batch(0)
    per_step = max(1, min(B, threads))
    sample = f"{per_step} of the 128 C4 utterances per step (full length 500), float64 oracle, OpenMP over utterances"
    times = []
    for i in range(args.warmup + args.steps):
        lo = (i * per_step) % B
        sub = type(w)(w.name, per_step, N, D, w.lengths[lo:lo + per_step], w.emis[lo:lo + per_step], den=w.den,
                      nums=w.nums[lo:lo + per_step])
        _, dt = cpu_oracle_rate(sub, per_step, threads)
        if i >= args.warmup:
            times.append(dt)
    frames = per_step * N
    value = frames * len(times) / sum(times)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "seq-frames/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / len(times),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD + " (sampled)", "global_batch": per_step, "seq_len": N,
                       "parallelism": "cpu-openmp"},
            "cpu_baseline": {"value": value, "unit": "seq-frames/s", "cores": threads, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": value, "unit": "seq-frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------- our arm

def ncu_traffic(args, n_launch: int):
    """DRAM bytes (read + write) of the den kernels of ONE step, measured live by ncu on
    a child process of this script (same build, same inputs, one lfmmi_loss_grad /
    fb_forward+fb_backward call): {kernel label: bytes per launch}.  None (with the
    reason) when ncu is not available or fails; never part of the timed region."""
    ncu = shutil.which("ncu") or "/usr/local/cuda/bin/ncu"
    if not os.path.exists(ncu):
        return None, "ncu not found"
    pat = "regex:^k_fbc?$"
    cmd = [ncu, "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum", "--clock-control",
           "none", "-k", pat, "-c", str(n_launch), "--csv", sys.executable, os.path.abspath(__file__),
           "--ncu-child", "--workload", args.workload]
    try:
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=300)
    except Exception as e:  # noqa: BLE001
        return None, f"ncu failed: {e}"
    rows = [ln for ln in r.stdout.splitlines() if ln.startswith('"')]
    if not rows:
        return None, f"ncu rc={r.returncode}: {r.stderr.strip()[-200:]}"
    per = {}
    for row in csv.DictReader(io.StringIO("\n".join(rows))):
        key = (row["ID"], row["Kernel Name"])
        v = float(row["Metric Value"].replace(",", ""))
        unit = row.get("Metric Unit", "")
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(unit, 1)
        d = per.setdefault(key, {"bytes": 0.0})
        if row["Metric Name"].startswith("dram__bytes"):
            d["bytes"] += v * scale
    out = {}
    for (_, kname), d in sorted(per.items(), key=lambda x: int(x[0][0])):
        kname = kname.split(" ", 1)[1] if kname.startswith("void ") else kname  # ncu prints "void k_fbc<…>(FBArgs)"
        label = ("k_fbc" if kname.startswith("k_fbc") else "k_fb") + ("_bwd[G=1]" if "<true" in kname or "<1" in kname
                                                                      else "_fwd[G=1]")
        out.setdefault(label, d["bytes"])
        out.setdefault(label.replace("[G=1]", "[G=B]"), d["bytes"])
    return out, "ncu (live: child process of this run, --metrics dram__bytes_read.sum,dram__bytes_write.sum)"


def ncu_child(args):
    """One call of the timed step on cuda:0 (profiled by the parent's ncu; no output)."""
    import torch

    import paper_2112_00709_b200 as fbx
    from paper_2112_00709_b200 import synth

    torch.cuda.set_device(0)
    w = make_batch(0, 1, args.workload)
    den = fbx.Graph.from_host(w.den)
    emis = torch.from_numpy(w.emis).cuda()
    lens = torch.from_numpy(w.lengths).cuda()
    if args.workload in ("c3", "c2"):
        logZ, alpha, _, st = fbx.fb_forward(den, emis, lens)
        fbx.fb_backward(den, emis, lens, alpha=alpha, status=st)
    else:
        num = fbx.Graph.from_host(synth.compose(w.nums))
        fbx.lfmmi_loss_grad(num, den, emis, lens)
    torch.cuda.synchronize()


def run_ours(args, rank, world, local):
    import torch
    import torch.distributed as dist

    import paper_2112_00709_b200 as fbx
    from paper_2112_00709_b200 import build, synth

    build.build()
    if world != args.gpus:
        log(f"[rank {rank}] note: --gpus {args.gpus} but WORLD_SIZE={world}; reporting n_gpus={world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    t0 = time.time()
    w = make_batch(rank, world, args.workload)
    Bw, Nw = w.B, w.N_max
    c3 = args.workload in ("c3", "c2")  # public fb_forward + fb_backward (fused state posteriors)
    vit = args.workload.startswith("viterbi")
    num = None if (c3 or vit) else fbx.Graph.from_host(synth.compose(w.nums))
    den = fbx.Graph.from_host(w.den)
    log(f"[rank {rank}] inputs ready in {time.time() - t0:.1f}s; den {den.info} num K_tot {num.K_tot if num else 0}")
    emis = torch.from_numpy(w.emis).to(dev)
    lens = torch.from_numpy(w.lengths).to(dev)
    loss = torch.empty(Bw, dtype=torch.float64, device=dev)
    totals = torch.empty(5, dtype=torch.float64, device=dev)
    status = torch.empty(Bw, dtype=torch.int32, device=dev)
    if vit:
        # N1: tropical-semiring best path (fb_viterbi) over the shared den graph
        L = fbx.lib()
        sp = fbx._dev
        score = torch.empty(Bw, dtype=torch.float64, device=dev)
        path = torch.empty((Bw, Nw), dtype=torch.int32, device=dev)
        vws = torch.empty(int(L.fb_viterbi_workspace_bytes(den.handle, Bw, Nw)), dtype=torch.uint8, device=dev)

        def step():
            fbx._check(L.fb_viterbi(den.handle, sp(emis, torch.float32, "emis"), sp(lens, torch.int32, "lengths"), Bw,
                                    Nw, sp(score, torch.float64, "score"), sp(path, torch.int32, "path"),
                                    sp(status, torch.int32, "status"), sp(vws, torch.uint8, "ws"), vws.numel(),
                                    fbx._stream()), "fb_viterbi")
            if world > 1:
                totals[0:1].copy_(score.sum().unsqueeze(0))
                dist.all_reduce(totals)
    elif c3:
        # fb_forward + fb_backward with fused state posteriors (SURVEY §8(d) C3 call sequence)
        alpha = torch.empty(den.lattice_numel(Bw, Nw), dtype=torch.float32, device=dev)
        ascale = torch.empty((Bw, Nw), dtype=torch.float64, device=dev)
        post = torch.empty(den.lattice_numel(Bw, Nw), dtype=torch.float32, device=dev)
        logZ = torch.empty(Bw, dtype=torch.float64, device=dev)
        logZb = torch.empty(Bw, dtype=torch.float64, device=dev)
        L = fbx.lib()
        sp = fbx._dev  # marshalling helper of the binding (pointer of a CUDA tensor)

        def step():
            s_ = fbx._stream()
            fbx._check(L.fb_forward(den.handle, sp(emis, torch.float32, "emis"), sp(lens, torch.int32, "lengths"), Bw,
                                    Nw, sp(alpha, torch.float32, "alpha"), sp(ascale, torch.float64, "scale"),
                                    sp(logZ, torch.float64, "logZ"), sp(status, torch.int32, "status"), s_),
                       "fb_forward")
            fbx._check(L.fb_backward(den.handle, sp(emis, torch.float32, "emis"), sp(lens, torch.int32, "lengths"),
                                     Bw, Nw, None, None, sp(logZb, torch.float64, "logZ_beta"),
                                     sp(alpha, torch.float32, "alpha"), sp(post, torch.float32, "post"), 0,
                                     sp(status, torch.int32, "status"), s_), "fb_backward")
            if world > 1:
                totals[0:1].copy_(logZ.sum().unsqueeze(0))
                dist.all_reduce(totals)
    else:
        grad = torch.empty_like(emis)
        ws = torch.empty(fbx.workspace_bytes(num, den, Bw, Nw), dtype=torch.uint8, device=dev)

        def step():
            fbx.lfmmi_loss_grad(num, den, emis, lens, grad, ws, loss, totals, status)
            if world > 1:
                dist.all_reduce(totals)  # NCCL on the current stream: Σ loss, Σ frames, Σ logZ, n_bad

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    st_host = status.cpu().numpy()
    assert (st_host == 0).all(), st_host
    # inputs smaller than L2 (the N2 shape: φ 30 MB) → flush L2 between timed steps
    # by writing a 256 MB scratch buffer outside the per-step event pairs
    flush = emis.numel() * 4 < 256 << 20
    scratch = torch.empty(64 << 20, dtype=torch.float32, device=dev) if flush else None
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    fbx.profile_reset()
    fbx.profile_enable(True)
    # one event pair per step (device time on the launching stream); without a flush
    # the steps run back to back and the whole-run time is first start → last end
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        for a_, b_ in evs:
            if flush:
                scratch.fill_(1.0)
            a_.record()
            step()
            b_.record()
        torch.cuda.synchronize()
    fbx.profile_enable(False)
    prof = fbx.profile_collect()
    per_step = [a_.elapsed_time(b_) for a_, b_ in evs]
    ms = sum(per_step) if flush else evs[0][0].elapsed_time(evs[-1][1])
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    fr = torch.tensor([float(w.lengths.sum())], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(fr)  # ranks' shards differ in C5
    frames_total = float(fr.item()) * args.steps
    value = frames_total / (ms / 1e3)

    # per-kernel roofline (dominant kernel: the denominator backward with the fused gradient epilogue)
    hbm, peak_src = measured_peaks()
    seq_frames = float(w.lengths.sum())
    Kw = w.den.K if hasattr(w.den, "K") else w.den.K_tot / w.B  # C2: mean states per numerator graph
    Dw = w.D if hasattr(w.den, "K") else min(w.D, Kw)          # C2: identity map, a graph reads K_b columns
    alg_bytes = {}  # algorithmic bytes per launch from the rank's true frames
    bp_bytes = 2 if Kw <= 32767 else 4
    alg_bytes["k_viterbi"] = seq_frames * (4 * min(Dw, Kw) + bp_bytes * Kw)  # φ row (the columns read) + backpointer row
    for kname in ("k_fb", "k_fbc"):
        if c3:  # backward: φ row + α̂ row in, γ row out; forward: φ row in, α̂ row out
            alg_bytes[kname + "_bwd[G=1]"] = seq_frames * (4 * Dw + 4 * Kw + 4 * Kw)
        else:   # backward: φ row + α̂ row in, grad row out; padded frames' grad rows are written 0 (fb.h)
            alg_bytes[kname + "_bwd[G=1]"] = seq_frames * (4 * Dw + 4 * Kw + 4 * Dw) + (Bw * Nw - seq_frames) * 4 * Dw
        alg_bytes[kname + "_fwd[G=1]"] = seq_frames * (4 * Dw + 4 * Kw)
    for k in list(alg_bytes):  # per-sequence graph batches (C2) launch the same kernels as "[G=B]"
        if k.endswith("[G=1]"):
            alg_bytes[k.replace("[G=1]", "[G=B]")] = alg_bytes[k]
    kern = {}
    for name, (cnt, tot_ms) in prof.items():
        avg = tot_ms / max(cnt, 1)
        kern[name] = {"launches": cnt, "avg_ms": avg}
        if name.startswith(("k_fb_", "k_fbc_")):
            kern[name]["frame_step_us"] = avg * 1e3 / Nw  # per-frame step latency of the recursion
        if name in alg_bytes:
            kern[name]["achieved_gbs"] = alg_bytes[name] / (avg / 1e3) / 1e9
    dom = max((k for k in kern if k in alg_bytes), key=lambda k: kern[k]["avg_ms"] * kern[k]["launches"])
    achieved = kern.get(dom, {}).get("achieved_gbs")
    roofline = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": hbm, "unit": "GB/s",
                "frac": (achieved / hbm) if achieved else None, "traffic": None, "peak_source": peak_src,
                "algorithmic_bytes_per_launch": alg_bytes[dom]}
    step_bytes = alg_bytes["k_viterbi"] if vit else alg_bytes["k_fb_bwd[G=1]"] + alg_bytes["k_fb_fwd[G=1]"]
    if args.workload == "c2":  # latency-bound: the per-frame step is the number to read
        roofline["bound"] = "latency"
    den_kind = "k_fbc (cluster)" if den.info["cluster_C"] else "k_fb (one CTA per sequence)"
    launches = sum(c for c, _ in prof.values())

    # end to end through the public API with host buffers (pinned φ in, totals + loss out)
    e2e = None
    if not (c3 or vit):
        emis_h = torch.from_numpy(w.emis).pin_memory()
        lens_h = torch.from_numpy(w.lengths).pin_memory()
        bufs = {}
        for _ in range(2):
            fbx.lfmmi_loss_grad_host(num, den, emis_h, lens_h, bufs)
        torch.cuda.synchronize()
        k2 = max(3, min(args.steps, 10))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for cs_ in bufs["copy_streams"]:
            cs_.wait_event(e0)  # the first upload starts inside the timed region
        for _ in range(k2):
            out = fbx.lfmmi_loss_grad_host(num, den, emis_h, lens_h, bufs)
            if world > 1:
                dist.all_reduce(bufs["totals"])
        e1.record()
        torch.cuda.synchronize()
        ems = e0.elapsed_time(e1)
        if world > 1:
            t = torch.tensor([ems], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t.item())
        e2e = {"value": float(fr.item()) * k2 / (ems / 1e3), "unit": "seq-frames/s",
               "h2d_bytes_per_step": int(emis_h.numel() * 4 + lens_h.numel() * 4),
               "d2h_bytes_per_step": int(out.numel() * 8), "steps": k2}

    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if rank != 0:
        return
    if not args.no_ncu and not vit:
        tr, src = ncu_traffic(args, 2)
        roofline["traffic_source"] = src
        if tr and dom in tr:
            roofline["traffic"] = tr[dom]
            roofline["traffic_ratio"] = tr[dom] / alg_bytes[dom]
    cpu = None
    if not args.no_cpu_baseline and not (c3 or vit):
        threads = len(os.sched_getaffinity(0))
        n_utts = max(1, min(w.B, 2 * threads))
        rate, dt = cpu_oracle_rate(w, n_utts, threads)
        cpu = {"value": rate, "unit": "seq-frames/s", "cores": threads, "kind": "oracle",
               "sample": f"{n_utts} of the {w.B} {w.name} utterances at full length ({w.N_max} frames), "
                         f"float64 C oracle, {dt:.1f} s wall"}
    line = {
        "metric": METRIC, "value": value, "unit": "seq-frames/s", "n_gpus": world, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": ms / args.steps, "higher_is_better": True,
        "step_ms": {"median": statistics.median(per_step), "min": min(per_step), "max": max(per_step),
                    "note": "per-step CUDA events of rank 0" + ("" if flush else " (steps back to back)")},
        "scaling": "strong" if args.workload == "c5-strong" else "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded; SURVEY §8(d) recipes)",
        "config": {"workload": {"c4": WORKLOAD, "paper": WORKLOAD_N2, "c3": WORKLOAD_C3,
                                "c2": "C2: 64 left-to-right numerator graphs (K 100-300, G = B), fb_forward + fb_backward "
                                      "with state posteriors, φ[64,180,300], N_b ~ U[max(120, L), 180]",
                                "viterbi": "N1: Viterbi (tropical semiring, fb_viterbi) over the C3 den, φ[128,500,3000]",
                                "viterbi-paper": "N1: Viterbi over the paper's Table 1 den (3022 st / 50,984 arcs, "
                                                 "schedule streamed from L2), φ[128,700,84]"}.get(args.workload,
                   f"{args.workload.upper()}: 1024-utterance pool, N_b log-normal median 250 in [50,700], LPT-sharded"),
                   "global_batch": Bw * world if args.workload != "c5-strong" else 1024, "seq_len": Nw,
                   "parallelism": f"dp{world}", "den_kernel": den_kind,
                   "l2": ("L2 flushed between timed steps (256 MB write outside the step events)" if flush else
                          "inputs larger than L2 (φ ≥ 512 MB, α̂ 768 MB per step)")},
        "hbm_fraction_of_step": (step_bytes / (ms / args.steps / 1e3) / 1e9) / hbm,
        "roofline": roofline, "kernels": kern, "gpu_launches": launches, "clocks": clk.summary(),
        "e2e": e2e, "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)


def spawn_ranks(args) -> int:
    """--gpus N > 1 outside a torchrun environment: start N ranks (one process per
    GPU) with torch.distributed.run on 127.0.0.1 and return their exit code."""
    if args.impl == "ours":
        import torch

        have = torch.cuda.device_count()
        if have < args.gpus:
            log(f"bench.py: --gpus {args.gpus} but only {have} CUDA device(s) visible")
            return 2
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-ncu", action="store_true", help="skip the live ncu DRAM-traffic capture (roofline.traffic)")
    ap.add_argument("--ncu-child", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--workload", default="c4",
                    choices=["c4", "c3", "c2", "c5-weak", "c5-strong", "paper", "viterbi", "viterbi-paper"],
                    help="c4 = the BASELINE metric config (default); c3 = den fwd+bwd+posteriors call sequence; "
                         "c5-* = variable-length 1024-utterance pool; paper = N2, the paper's Table 1 graph shape")
    args = ap.parse_args()
    if args.ncu_child:
        ncu_child(args)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_ours(args, rank, world, local)


if __name__ == "__main__":
    main()
