"""Benchmark: TimelyFreeze pipeline training step on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--model llama-8b]

Workload (BASELINE.json configs[2], the north-star configuration): LLaMA-3-8B-shaped decoder
(h 4096, 32 layers, GQA 32/8, head_dim 128, vocab 128256), 1F1B, PP = N, M = 32 microbatches of
2 x 2048 tokens, synthetic uniform tokens and N(0, 0.02) random-init weights. N = 1: one stage holds
all 32 layers (the whole model fits one B200's HBM). --gpus N > 1 without a launcher spawns the N
ranks itself (torch.distributed.run on 127.0.0.1).

Procedure (ours): run the Alg. 1 controller untimed through warm-up, the two monitoring halves
(CUDA-event action times), the LP solve at T_m and the AFR ramp, then W stable-phase warm-up
steps, then K timed stable-phase steps (device time, CUDA events on the trainer's stream, max over
ranks). The same steps are timed with every unit unfrozen (no-freeze) for the speed-up, and K
more end-to-end through the C-ABI with pinned host token buffers and the loss read back (e2e).

Reference arm (--impl reference) and cpu_baseline: the reference's own CPU implementation of the
path (oracle/_ref, the unmodified reference compiled here) at the FULL parameter count of the
workload, sharded element-wise over every host core: per step the controller work (schedule +
DAG + longest path + the step's S*M exact-count masks) and the per-parameter pass (apf_update +
the masked accumulation and SGD update of run_masked_sgd). Only steps actually timed are reported.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "tokens/sec per PP step at 1/2/4/8 B200 vs no-freeze; batch time vs LP makespan"


_T0 = time.perf_counter()


def progress(msg: str) -> None:
    """Phase marks on stderr (the JSON line stays the only stdout output)."""
    print(f"[bench {time.perf_counter() - _T0:7.1f}s] {msg}", file=sys.stderr, flush=True)


def dist_env():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("LOCAL_RANK", "0"))


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_{os.getpid()}.csv")

    def __enter__(self):
        os.makedirs(os.path.dirname(self.path), exist_ok=True)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                          "-lms", "200"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.f.close()

    def summary(self) -> dict:
        rows = []
        try:
            for line in open(self.path):
                p = [x.strip() for x in line.split(",")]
                if len(p) >= 9:
                    rows.append(p)
        except Exception:
            pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        load = [s for s in sm if s > 500] or sm
        reasons = set()
        for r in rows:
            for name, col in (("hw_slowdown", 5), ("hw_thermal_slowdown", 6), ("sw_thermal_slowdown", 7), ("sw_power_cap", 8)):
                if r[col].lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": float(rows[0][2]),
                "samples": len(rows), "reasons": sorted(reasons)}


def load_peaks() -> dict:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return {"hbm_gbs": p["hbm_gbs"], "bf16_tflops": p["bf16_tflops"],
                "bf16_tflops_sustained": p.get("bf16_tflops_sustained", p["bf16_tflops"]), "source": "measured"}
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "source": "fallback"}


def step_flops(shape, M: int, mean_ratio: float, S: int = 1) -> dict:
    """Algorithmic FLOPs of one step: matmul fwd 2TP, dX 2TP, dW (1-r) 2TP, causal attention fwd 2Tsh and bwd 5Tsh."""
    T = shape.tokens
    if getattr(shape, "family", 0) == 1:  # ViT: patch embedding on the patch rows, head on the cls rows
        B = shape.micro_batch
        mm = 2 * T * shape.layers * shape.matmul_params_per_layer() + 2 * B * (shape.seq - 1) * shape.hidden * \
            shape.patch_dim + 2 * B * shape.vocab * shape.hidden
        attn_f = 4.0 * T * shape.seq * shape.n_heads * shape.head_dim * shape.layers  # bidirectional
    else:
        P = shape.layers * shape.matmul_params_per_layer() + shape.vocab * shape.hidden
        mm = 2 * T * P
        attn_f = 2.0 * T * shape.seq * shape.n_heads * shape.head_dim * shape.layers  # causal: half of 4Tsh
    attn_b = 2.5 * attn_f
    return {"fwd": M * (mm + attn_f), "dx": M * (mm + attn_b), "dw": M * mm * (1.0 - mean_ratio)}


def gemm_roofline(peaks: dict, shape, launches: int, total_ms: float) -> dict:
    """Dominant kernel: the K1 tcgen05 CTA-pair GEMM of the gate|up projection (the largest
    per-layer GEMM), its launches inside the timed steps bracketed with CUDA events on the
    trainer's stream (pf_probe_*). achieved = algorithmic FLOPs per launch / mean duration;
    traffic = DRAM bytes per launch from the committed ncu --set full capture of this kernel."""
    vit = getattr(shape, "family", 0) == 1
    T, h, N = shape.tokens, shape.hidden, shape.ffn if vit else 2 * shape.ffn
    if launches <= 0 or total_ms <= 0:
        return {"bound": "tensor", "kernel": None, "achieved": None, "peak": peaks["bf16_tflops"], "unit": "TFLOP/s",
                "frac": None, "traffic": None, "note": "probe saw no launches"}
    ms = total_ms / launches
    flops = 2.0 * T * N * h
    achieved = flops / (ms * 1e-3) / 1e12
    fused = os.environ.get("PF_FUSE_SWIGLU", "") != "0"
    kernel = f"gemm_tcgen05_pair (cta_group::2) fwd {T}x{N}x{h} (K1, {'fc1' if vit else 'gate|up'}" + \
        ((", bias + GELU" if vit else ", SwiGLU") + " fused in the epilogue)" if fused else ")")
    # the kernel is timed inside the long timed steps, so the roofline is the SUSTAINED bf16 peak
    # (cuBLAS back to back, power-capped clocks); the burst figure is reported beside it
    sus, burst = peaks["bf16_tflops_sustained"], peaks["bf16_tflops"]
    return {"bound": "tensor", "kernel": kernel, "achieved": round(achieved, 1),
            "peak": sus, "unit": "TFLOP/s", "frac": round(achieved / sus, 4),
            "traffic": ncu_traffic(kernel), "avg_launch_ms": round(ms, 4), "launches_timed": launches,
            "algorithmic_flop_per_launch": flops, "peak_source": peaks["source"],
            "peak_kind": "sustained (kernel timed inside the step)", "burst_peak": burst,
            "frac_of_burst": round(achieved / burst, 4)}


def ncu_traffic(kernel: str):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel` from profiles/roofline_traffic.json
    (written by tools/ncu_traffic.py from an ncu --set full capture of this bench command), else None."""
    path = os.path.join(ROOT, "profiles", "roofline_traffic.json")
    try:
        with open(path) as f:
            d = json.load(f)
        for e in d if isinstance(d, list) else [d]:  # one entry per config's roofline kernel
            if e.get("kernel") == kernel:
                return e["bytes_per_launch"]
        return None
    except (OSError, ValueError, KeyError):
        return None


# ---------------------------------------------------------------- reference CPU path (oracle/_ref)
# Only the reference arm and the cpu_baseline leg import oracle/ (the checker), never the product.
_RW_MASKS = None


def _ref_worker_init(masks):
    global _RW_MASKS
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    _RW_MASKS = masks


def _ref_worker_pass(job):
    import ref  # noqa: E402  (oracle, reference arm / cpu_baseline only)

    begin, end, block, per_unit = job
    return ref.param_pass_seconds(begin, end, block, _RW_MASKS, per_unit)


class ReferenceCpuStep:
    """One step of this workload through the reference's CPU implementation (oracle/_ref), at the
    full parameter count, on `workers` processes (element-wise shards of the parameters):

      controller (main process): build_schedule + build_dag + longest_path_start_times and the
        step's S*M exact-count masks over the stage's units (run_freezing_masks, freezectl.cpp:185-211);
      per-parameter pass (workers): apf_update (freezectl.cpp:147-156) and the masked accumulation
        sum_m U_m (.) g + SGD update (run_masked_sgd, sandbox.cpp:232-250) over every parameter.

    Step time = controller + the slowest worker's pass (wall clock around both)."""

    BLOCK = 1 << 16

    def __init__(self, kind: str, R: int, C: int, M: int, n_units: int, n_params: int, ratio: float,
                 workers: int | None = None):
        import multiprocessing as mp

        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import ref  # noqa: E402  (oracle, reference arm / cpu_baseline only)

        if not ref.available():
            raise RuntimeError("oracle/_ref/libpfref.so is not built")
        self.ref = ref
        self.kind, self.R, self.C, self.M = kind, R, C, M
        self.n_units, self.n_params, self.ratio = n_units, n_params, ratio
        self.workers = workers or os.cpu_count() or 1
        _, masks = ref.controller_step(kind, R, C, M, n_units, ratio)
        per_unit = max(1, n_params // max(1, n_units))
        bounds = [n_params * i // self.workers for i in range(self.workers + 1)]
        self.jobs = [(bounds[i], bounds[i + 1], self.BLOCK, per_unit) for i in range(self.workers)]
        self.pool = mp.get_context("spawn").Pool(self.workers, initializer=_ref_worker_init, initargs=(masks,))
        self.seed = 42

    def step(self) -> dict:
        w0 = time.perf_counter()
        self.seed += 1
        ctl_s, _ = self.ref.controller_step(self.kind, self.R, self.C, self.M, self.n_units, self.ratio, self.seed)
        secs = self.pool.map(_ref_worker_pass, self.jobs, chunksize=1)
        wall = time.perf_counter() - w0
        return {"wall_s": wall, "controller_s": ctl_s, "param_pass_s": max(secs)}

    def describe(self) -> str:
        S = self.R * self.C
        return (f"reference CPU step at full size: controller (schedule + DAG + longest path + {S * self.M} "
                f"sample_mask over {self.n_units:,} units) + apf_update and masked SGD over all "
                f"{self.n_params:,} parameters at frozen ratio {self.ratio:.3f}, {self.workers} worker processes "
                f"(element-wise shards, {self.BLOCK}-element blocks)")

    def close(self):
        self.pool.terminate()
        self.pool.join()


def _workload_params(shape, S: int) -> tuple[int, int]:
    """(parameters of the whole job, freeze units of stage 1): the same counts both arms report."""
    from paper_2602_05754_b200.engine import param_layout

    n_params = sum(param_layout(shape, s, S)["n_params"] for s in range(1, S + 1))
    return n_params, param_layout(shape, 1, S)["n_units"]


def run_reference(args) -> None:
    rank, world, _ = dist_env()
    if rank != 0:
        return
    shape = model_shape(args)
    M = args.microbatches
    C = stages_per_rank(args)
    S = args.gpus * C
    n_params, units = _workload_params(shape, S)
    ratio = args.r_max  # the LP's stable-phase mean freeze ratio is r_max on these workloads
    cpu = ReferenceCpuStep(args.schedule, args.gpus, C, M, units, n_params, ratio)
    budget = float(os.environ.get("PF_REF_BUDGET_S", "150"))
    try:
        warm = min(args.warmup, 1)
        for _ in range(warm):
            cpu.step()
        timed = []
        t0 = time.perf_counter()
        for _ in range(args.steps):
            timed.append(cpu.step())
            if time.perf_counter() - t0 > budget:
                break
    finally:
        cpu.close()
    step_s = statistics.mean(r["wall_s"] for r in timed)
    tokens = M * shape.tokens
    value = tokens / step_s
    line = {"impl": "reference", "metric": METRIC, "value": round(value, 2), "unit": "tokens/s", "n_gpus": args.gpus,
            "steps": len(timed), "steps_requested": args.steps, "warmup": warm, "warmup_requested": args.warmup,
            "ms_per_step": round(step_s * 1e3, 3), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": _config(args, shape),
            "cpu_baseline": {"value": round(value, 2), "unit": "tokens/s", "cores": cpu.workers, "kind": "reference",
                             "sample": cpu.describe()},
            "e2e": {"value": round(value, 2), "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "n_params": n_params, "nproc": os.cpu_count(),
            "step_breakdown_s": {"controller": round(statistics.mean(r["controller_s"] for r in timed), 4),
                                 "param_pass": round(statistics.mean(r["param_pass_s"] for r in timed), 3)},
            "timed_budget_s": budget,
            "note": ("the reference has no transformer math; its step is the CPU path of the freeze controller, "
                     "APF metric and masked update at the workload's parameter count. Steps stop early (reported "
                     "'steps') once the timed steps exceed timed_budget_s.")}
    print(json.dumps(line), flush=True)


def model_shape(args):
    """The preset of --model, with --layers overriding the layer count (a per-rank slice of a
    pipeline that does not fit one GPU, e.g. LLaMA-13B's 5 layers per rank at PP=8)."""
    import dataclasses

    from paper_2602_05754_b200.engine import PRESETS

    shape = PRESETS[args.model]
    return dataclasses.replace(shape, layers=args.layers) if args.layers else shape


def _units_for(shape, S: int) -> int:
    from paper_2602_05754_b200.engine import param_layout

    return param_layout(shape, S, S)["n_units"] if S >= 1 else 0


def _config(args, shape) -> dict:
    cfg_idx = {"llama-1b": 1, "llama-8b": 2, "llama-13b": 3, "vit-l-32": 4}.get(args.model)
    tag = f"BASELINE configs[{cfg_idx}] shapes" if cfg_idx is not None else "test shapes"
    if getattr(args, "layers", 0):
        tag += f", {args.layers}-layer slice"
    return {"workload": f"{args.model}-shaped {args.schedule} PP={args.gpus} ({tag})",
            "model": args.model, "hidden": shape.hidden, "layers": shape.layers, "ffn": shape.ffn,
            "heads": shape.n_heads, "kv_heads": shape.n_kv_heads, "vocab": shape.vocab,
            "global_batch": args.microbatches * shape.micro_batch, "seq_len": shape.seq,
            "microbatches": args.microbatches, "micro_batch": shape.micro_batch, "schedule": args.schedule,
            "parallelism": f"pp{args.gpus}", "stages_per_rank": stages_per_rank(args), "r_max": args.r_max,
            "phases": list(args.phases),
            "optimizer": args.optimizer,
            "l2": "inputs larger than L2 (>2 GB of weights and activations touched per step)"}


def stages_per_rank(args) -> int:
    """Virtual stages per GPU: 2 for the V-shaped zbv / zbv-split, --chunks for interleaved."""
    if args.schedule in ("zbv", "zbv-split"):
        return 2
    return args.chunks if args.schedule in ("interleaved-1f1b", "interleaved") else 1


def _dev_view(ptr: int, n: int, dtype):
    """Zero-copy torch view of a device buffer returned by the C-ABI."""
    import torch

    typestr = {torch.float32: "<f4", torch.bfloat16: "<i2"}[dtype]
    obj = type("Cai", (), {})()
    obj.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False), "version": 3}
    t = torch.as_tensor(obj, device="cuda")
    return t.view(torch.bfloat16) if dtype is torch.bfloat16 else t


def pp_consistency_check(world: int, rank: int, local: int) -> dict:
    """Before timing: one step of a tiny LLaMA pipeline split over the job's ranks (PP = N, NCCL P2P)
    against the same model as ONE stage on this GPU, on identical weights and tokens, nothing frozen.
    The PP = 1 copy is assembled from every rank's stage parameters (all-gathered), so both compute
    the same function; the per-parameter update must agree (max relative difference over ranks).
    At N = 1 the split is 2 local stages on this GPU (same mapping code, no NCCL)."""
    import dataclasses

    import numpy as np
    import torch

    from paper_2602_05754_b200.engine import PRESETS, Trainer, param_layout

    split = max(2, world)
    shape = dataclasses.replace(PRESETS["tiny"], layers=max(4, split))
    M, lr = 4, 0.5
    if world > 1:
        import torch.distributed as dist

        trA = Trainer(shape, "1f1b", world, 1, M, rank=rank, lr=lr, seed=3, device=local)
        trA.init_comm()
        stages = [rank + 1]
    else:
        trA = Trainer(shape, "interleaved-1f1b", 1, 2, M, rank=0, lr=lr, seed=3, device=local)
        stages = [1, 2]
    trB = Trainer(shape, "1f1b", 1, 1, M, rank=0, lr=lr, seed=3, device=local)
    trA.set_override(0.0)
    trB.set_override(0.0)
    layB = param_layout(shape, 1, 1)
    offB = {e["name"]: e for e in layB["units"] + layB["dense"]}
    bufB = trB.stage_buffers(0)
    mB = _dev_view(bufB["master"], bufB["n_params"], torch.float32)
    wB = _dev_view(bufB["weights"], bufB["n_params"], torch.bfloat16)

    def stage_master(i):
        b = trA.stage_buffers(i)
        return _dev_view(b["master"], b["n_params"], torch.float32)

    # every stage's master parameters, gathered to every rank
    mine = {s: stage_master(i).clone() for i, s in enumerate(stages)}
    if world > 1:
        n_max = max(param_layout(shape, s, split)["n_params"] for s in range(1, split + 1))
        pad = torch.zeros(n_max, device="cuda")
        pad[: mine[rank + 1].numel()] = mine[rank + 1]
        parts = [torch.zeros_like(pad) for _ in range(world)]
        dist.all_gather(parts, pad)
        allm = {s + 1: parts[s] for s in range(world)}
    else:
        allm = mine
    before = {}
    for s in range(1, split + 1):
        lay = param_layout(shape, s, split)
        for e in lay["units"] + lay["dense"]:
            n = e["rows"] * e["cols"]
            dst = offB[e["name"]]["offset"]
            mB[dst:dst + n] = allm[s][e["offset"]:e["offset"] + n]
            wB[dst:dst + n] = mB[dst:dst + n].bfloat16()
            if s in stages:
                before[e["name"]] = (s, e)
    torch.cuda.synchronize()
    rng = np.random.default_rng(123)
    tok = rng.integers(0, shape.vocab, size=(M, shape.tokens), dtype=np.int32)
    tgt = rng.integers(0, shape.vocab, size=(M, shape.tokens), dtype=np.int32)
    thetaB0 = mB.clone()
    thetaA0 = {s: stage_master(i).clone() for i, s in enumerate(stages)}
    rA = trA.step(1, tok, tgt)
    rB = trB.step(1, tok, tgt)
    torch.cuda.synchronize()
    worst, bitwise = 0.0, True
    for name, (s, e) in before.items():
        i = stages.index(s)
        n = e["rows"] * e["cols"]
        dA = stage_master(i)[e["offset"]:e["offset"] + n] - thetaA0[s][e["offset"]:e["offset"] + n]
        o = offB[name]["offset"]
        dB = mB[o:o + n] - thetaB0[o:o + n]
        bitwise &= bool(torch.equal(dA, dB))
        den = dB.norm().item()
        if den > 0:
            worst = max(worst, (dA - dB).norm().item() / den)
    if world > 1:
        t = torch.tensor([worst, 0.0 if bitwise else 1.0], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        worst, bitwise = t[0].item(), t[1].item() == 0.0
    trA.close()
    trB.close()
    return {"what": f"tiny LLaMA ({shape.layers} layers, M={M}) split over {split} stages "
                    f"({'NCCL P2P over ' + str(world) + ' ranks' if world > 1 else '2 local stages, 1 GPU'}) vs 1 stage",
            "max_rel_update_diff": worst, "bitwise_equal": bitwise, "ok": worst <= 1e-2,
            "loss_pp1": round(rB["loss"], 6)}


def run_ours(args) -> None:
    import numpy as np
    import torch

    from paper_2602_05754_b200 import _native
    from paper_2602_05754_b200.engine import PRESETS, Trainer

    rank, world, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        # NCCL init logging (communicator ranks / transports) for the run's record
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("nccl")
    progress("pp consistency check")
    pp_check = pp_consistency_check(world, rank, local)
    progress(f"pp check done: {pp_check['max_rel_update_diff']:.2e}")
    shape = model_shape(args)
    M = args.microbatches
    phases = tuple(args.phases)
    C = stages_per_rank(args)
    tr = Trainer(shape, args.schedule, world, C, M, rank=rank, phases=phases, r_max=args.r_max, lr=1e-4,
                 seed=args.seed, device=local, optimizer=args.optimizer, weight_decay=0.1 if args.optimizer == "adamw" else 0.0)
    lib = _native.device()
    if world > 1:
        tr.init_comm()
    stream = torch.cuda.ExternalStream(lib.pf_trainer_stream(tr._ctx))
    tokens_per_step = M * shape.tokens

    # ---- controller: warm-up, monitoring, LP solve, ramp (untimed)
    t = 0
    ctl = []
    progress("trainer ready; controller steps")
    for t in range(1, phases[2] + 1):
        ctl.append(tr.step(t))
        progress(f"controller step {t}: loss {ctl[-1]['loss']:.4f} batch {ctl[-1]['batch_ms']:.1f} ms")
    plan = tr.get_plan()

    def timed_steps(start_t: int, k: int, host=None):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        res = []
        c0 = lib.pf_device_launch_count()
        e0.record(stream)
        w0 = time.perf_counter()
        for i in range(k):
            if host is not None:
                res.append(tr.step(start_t + i, host[0], host[1]))
            else:
                res.append(tr.step(start_t + i))
        e1.record(stream)
        torch.cuda.synchronize()
        wall = time.perf_counter() - w0
        launches = lib.pf_device_launch_count() - c0
        return e0.elapsed_time(e1), wall, res, launches

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        import torch.distributed as dist

        v = torch.tensor([x], device="cuda")
        dist.all_reduce(v, op=dist.ReduceOp.MAX)
        return v.item()

    # ---- stable freeze: warm-up then timed
    t = phases[2] + 1
    for i in range(args.warmup):
        tr.step(t + i)
    t += args.warmup
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    progress("timed freeze steps")
    lib.pf_probe_enable(1)  # time the dominant kernel's launches inside the timed steps
    ncu_range = bool(os.environ.get("PF_NCU_RANGE"))  # ncu --profile-from-start off: the timed steps only
    if ncu_range:
        torch.cuda.profiler.start()
    with ClockSampler(local) as clk:
        dev_ms, wall_s, res, launches = timed_steps(t, args.steps)
    if ncu_range:
        torch.cuda.profiler.stop()
    probe_n, probe_ms = ctypes.c_int(0), ctypes.c_double(0.0)
    _native.check(lib.pf_probe_read(ctypes.byref(probe_n), ctypes.byref(probe_ms)), "pf_probe_read")
    lib.pf_probe_enable(0)
    t += args.steps
    dev_ms = max_over_ranks(dev_ms)
    ms_step = dev_ms / args.steps
    value = tokens_per_step / (ms_step * 1e-3)

    # ---- no-freeze comparison (every unit updated; a shorter run: it is the speed-up's denominator)
    nf_steps = min(args.steps, 8)
    progress(f"freeze {ms_step:.1f} ms/step; no-freeze steps")
    tr.set_override(0.0)
    for i in range(2):
        tr.step(t + i)
    t += 2
    nf_ms, _, nf_res, _ = timed_steps(t, nf_steps)
    t += nf_steps
    nf_ms = max_over_ranks(nf_ms) / nf_steps
    tr.set_override(None)

    # ---- e2e through the C-ABI with host (pinned) token buffers; loss read back each step. The
    # host tokens are drawn from one seeded stream, identical on every rank (the first stage's
    # tokens and the last stage's targets then belong to the same microbatches).
    T = shape.tokens
    g = torch.Generator().manual_seed(args.seed)
    host_tok = torch.randint(0, shape.vocab, (M, T), dtype=torch.int32, generator=g).pin_memory()
    host_tgt = torch.randint(0, shape.vocab, (M, T), dtype=torch.int32, generator=g).pin_memory()
    hp = (host_tok.numpy(), host_tgt.numpy())
    progress(f"no-freeze {nf_ms:.1f} ms/step; e2e steps")
    e2e_dev, e2e_wall, e2e_res, _ = timed_steps(t, args.steps, host=hp)
    progress("e2e done")
    t += args.steps
    e2e_wall = max_over_ranks(e2e_wall)
    words = sum(((tr.stage_buffers(i)["n_units"] + 63) // 64 + 1) for i in range(tr.info["local_stages"])) * M
    h2d = 2 * M * T * 4 + words * 8

    peaks = load_peaks() if rank == 0 else None
    if rank == 0:
        mean_ratio = statistics.mean(r["mean_ratio"] for r in res)
        fl = step_flops(shape, M, mean_ratio)
        total_flops = sum(fl.values())
        batch_ms = statistics.mean(r["batch_ms"] for r in res)
        pred_ms = statistics.mean(r["predicted_ms"] for r in res)
        roof = gemm_roofline(peaks, shape, probe_n.value, probe_ms.value)
        cpu = {"value": None, "unit": "tokens/s", "cores": None, "kind": "reference", "sample": "not run (N > 1)"}
        if world == 1 and not os.environ.get("PF_SKIP_CPU_BASELINE"):
            # the reference's CPU path on this host's cores, one full-size step (after the timed region)
            n_params, units = _workload_params(shape, world * C)
            progress("cpu_baseline: one reference CPU step")
            try:
                ref_step = ReferenceCpuStep(args.schedule, world, C, M, units, n_params, mean_ratio)
                try:
                    r = ref_step.step()
                finally:
                    ref_step.close()
                cpu = {"value": round(tokens_per_step / r["wall_s"], 2), "unit": "tokens/s", "cores": ref_step.workers,
                       "kind": "reference", "sample": ref_step.describe() + " (1 step)",
                       "ms_per_step": round(r["wall_s"] * 1e3, 1)}
            except Exception as e:  # pragma: no cover - oracle missing on the box
                cpu["sample"] = f"unavailable: {e}"
        line = {
            "metric": METRIC, "value": round(value, 1), "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_step, 3), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic (uniform tokens, N(0,0.02) random-init weights)",
            "config": _config(args, shape),
            "nofreeze": {"value": round(tokens_per_step / (nf_ms * 1e-3), 1), "ms_per_step": round(nf_ms, 3),
                         "steps": nf_steps},
            "freeze_speedup": round(nf_ms / ms_step, 4),
            "batch_vs_lp": {"batch_ms": round(batch_ms, 3), "lp_makespan_ms": round(pred_ms, 3),
                            "ratio": round(batch_ms / pred_ms, 4) if pred_ms else None,
                            "plan_makespan_base_ms": round(plan["makespan_base"], 3) if plan else None,
                            "plan_makespan_opt_ms": round(plan["makespan_opt"], 3) if plan else None,
                            "plan_mean_ratio": round(float(plan["ratios"].mean()), 4) if plan else None,
                            "lp_solve_ms": round(tr.get_info()["lp_solve_ms"], 3)},
            "realised_frozen_fraction": round(mean_ratio, 4),
            "step_tflops": round(total_flops / (ms_step * 1e-3) / 1e12, 1),
            "mfu_of_measured_peak": round(total_flops / (ms_step * 1e-3) / 1e12 / peaks["bf16_tflops_sustained"], 4),
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": {"value": round(tokens_per_step * args.steps / e2e_wall, 1), "unit": "tokens/s",
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": 4},
            "clocks": clk.summary(),
            "gpu_launches": int(launches),
            "attention_backend": attention_backend(shape, lib),
            "loss": {"first": round(ctl[0]["loss"], 4), "last": round(res[-1]["loss"], 4)},
            "n_params": tr.info["params"] if world == 1 else None,
            "pp_check": pp_check,
        }
        print(json.dumps(line), flush=True)
    tr.close()
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


def attention_backend(shape, lib) -> str:
    """Which attention the step ran: ViT with S <= 64 and head_dim 64 uses the hand-written
    short-sequence kernel (vit_attention.cu) unless PF_VIT_ATTN=cudnn; everything else the
    library fused attention pf_attention_backend() names."""
    if getattr(shape, "family", 0) == 1 and shape.seq <= 64 and shape.head_dim == 64 and \
            os.environ.get("PF_VIT_ATTN") != "cudnn":
        return "vit_attn (own mma.sync kernel, S <= 64)"
    return lib.pf_attention_backend().decode()


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--model", default="llama-8b")
    ap.add_argument("--schedule", default="1f1b",
                    choices=["gpipe", "1f1b", "interleaved-1f1b", "zbv", "zbv-split"])
    ap.add_argument("--chunks", type=int, default=2, help="virtual stages per GPU for interleaved-1f1b")
    ap.add_argument("--microbatches", type=int, default=32)
    ap.add_argument("--layers", type=int, default=0,
                    help="override the preset's layer count (a per-rank slice of a larger pipeline)")
    ap.add_argument("--r-max", type=float, default=0.8)
    ap.add_argument("--phases", type=int, nargs=4, default=[1, 7, 8, 10000],
                    help="T_w T_m T_f T_total: warm-up 1, monitoring 2-6 (3 unfrozen + 2 frozen samples), LP at 7")
    ap.add_argument("--seed", type=int, default=42)
    ap.add_argument("--optimizer", choices=["sgd", "adamw"], default="sgd",
                    help="sgd = the reference's masked update (sandbox.cpp:250); adamw = the paper's optimizer")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # no launcher: spawn one rank per GPU on this node (same command line)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", os.environ.get("MASTER_PORT", "29531"),
               os.path.abspath(__file__), *sys.argv[1:]]
        raise SystemExit(subprocess.call(cmd))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
