"""Python handle on the device stage engine (libpf_device.so, include/pf_device.h).

`Trainer` drives Alg. 1 for one rank: schedule/DAG/LP/controller in the host C++
layer, the LLaMA-shaped stage step in hand-written sm_100a kernels. There is no
Python or CPU compute path: every method calls the native library.
"""
from __future__ import annotations

import ctypes
from dataclasses import asdict, dataclass

import numpy as np

from . import _native
from ._device_sigs import PfModelCfg, PfStepResult, PfTrainCfg, PfTrainerInfo
from .pipefreeze import KINDS, SPLIT_KINDS


@dataclass(frozen=True)
class ModelShape:
    hidden: int
    ffn: int
    n_heads: int
    n_kv_heads: int
    head_dim: int
    vocab: int
    layers: int
    seq: int
    micro_batch: int
    rope_theta: float = 500000.0
    norm_eps: float = 1e-5
    init_std: float = 0.02
    family: int = 0  # 0 LLaMA decoder, 1 ViT encoder (vocab = classes, micro_batch = images)
    image: int = 224
    patch: int = 32
    channels: int = 3

    @property
    def tokens(self) -> int:
        return self.seq * self.micro_batch

    @property
    def patch_dim(self) -> int:
        return self.patch * self.patch * self.channels

    @property
    def qkv_dim(self) -> int:
        return (self.n_heads + 2 * self.n_kv_heads) * self.head_dim

    def matmul_params_per_layer(self) -> int:
        h = self.hidden
        mlp_in = self.ffn if self.family == 1 else 2 * self.ffn
        return self.qkv_dim * h + h * self.n_heads * self.head_dim + mlp_in * h + h * self.ffn


PRESETS = {
    # unit tests / CPU-oracle parity (config 1 model step)
    "tiny": ModelShape(256, 512, 4, 2, 64, 1024, 4, 128, 2),
    # LLaMA-3.2-1B shapes (BASELINE configs[1]); untied LM head
    "llama-1b": ModelShape(2048, 8192, 32, 8, 64, 128256, 16, 2048, 2),
    # LLaMA-3-8B shapes (configs[2])
    "llama-8b": ModelShape(4096, 14336, 32, 8, 128, 128256, 32, 2048, 2),
    # LLaMA-2-13B shapes (configs[3])
    "llama-13b": ModelShape(5120, 13824, 40, 40, 128, 32000, 40, 2048, 1, rope_theta=10000.0),
    # ViT-L/32 (configs[4], C5): 224^2 / 32^2 patches -> 49 + cls = 50 tokens, 64 images per microbatch
    "vit-l-32": ModelShape(1024, 4096, 16, 16, 64, 1000, 24, 50, 64, norm_eps=1e-6, family=1),
    # small ViT for parity tests: 48^2 images, 16^2 patches -> 9 + cls = 10 tokens, 64 images (T = 640)
    "vit-tiny": ModelShape(256, 512, 4, 4, 64, 1000, 4, 10, 64, norm_eps=1e-6, family=1, image=48, patch=16),
}


def stage_layers(layers: int, S: int, s: int) -> tuple[int, int]:
    """Layers [begin, end) of 1-based stage s; the first L % S stages take one extra (trainer.cpp stage_spec)."""
    base, extra = divmod(layers, S)
    begin = (s - 1) * base + min(s - 1, extra)
    return begin, begin + base + (1 if s - 1 < extra else 0)


def param_layout(shape: ModelShape, s: int, S: int) -> dict:
    """Offsets of every parameter in a stage's flat buffers (mirror of Stage's constructor)."""
    align = 64
    off = 0
    out = {"units": [], "dense": []}

    def add(name, rows, cols, freezable):
        nonlocal off
        ent = dict(name=name, offset=off, rows=rows, cols=cols, freezable=freezable)
        off = (off + rows * cols + align - 1) // align * align
        (out["units"] if freezable else out["dense"]).append(ent)
        return ent

    b, e = stage_layers(shape.layers, S, s)
    h = shape.hidden
    if shape.family == 1:  # VitStage constructor order
        if s == 1:
            add("patch_w", h, shape.patch_dim, True)
        for layer in range(b, e):
            add(f"l{layer}.wqkv", 3 * h, h, True)
            add(f"l{layer}.wo", h, h, True)
            add(f"l{layer}.w1", shape.ffn, h, True)
            add(f"l{layer}.w2", h, shape.ffn, True)
        if s == S:
            add("head", shape.vocab, h, True)
        for layer in range(b, e):
            for name, n in (("bqkv", 3 * h), ("bo", h), ("b1", shape.ffn), ("b2", h), ("ln1g", h), ("ln1b", h),
                            ("ln2g", h), ("ln2b", h)):
                add(f"l{layer}.{name}", 1, n, False)
        if s == 1:
            add("patch_b", 1, h, False)
            add("cls", 1, h, False)
            add("pos", shape.seq, h, False)
        if s == S:
            add("lnfg", 1, h, False)
            add("lnfb", 1, h, False)
            add("headb", 1, shape.vocab, False)
        return _finish_layout(out, off)
    for layer in range(b, e):
        add(f"l{layer}.wqkv", shape.qkv_dim, h, True)
        add(f"l{layer}.wo", h, shape.n_heads * shape.head_dim, True)
        add(f"l{layer}.wgu", 2 * shape.ffn, h, True)
        add(f"l{layer}.wd", h, shape.ffn, True)
    if s == S:
        add("wlm", shape.vocab, h, True)
    for layer in range(b, e):
        add(f"l{layer}.g1", 1, h, False)
        add(f"l{layer}.g2", 1, h, False)
    if s == S:
        add("gf", 1, h, False)
    if s == 1:
        add("emb", shape.vocab, h, False)
    return _finish_layout(out, off)


def _finish_layout(out: dict, off: int) -> dict:
    u = 0
    for ent in out["units"]:
        ent["unit_offset"] = u
        ent["tiles_n"] = (ent["cols"] + 127) // 128
        ent["units"] = ((ent["rows"] + 127) // 128) * ent["tiles_n"]
        u += ent["units"]
    out["n_units"] = u
    out["n_params"] = off
    return out


def _check(rc: int, what: str) -> None:
    if rc != 0:
        lib = _native.device()
        msg = lib.pf_engine_last_error().decode() or lib.pf_device_last_error().decode()
        raise _native.PfError(rc, f"{what} failed with status {rc}: {msg}")


class Trainer:
    """One rank of the TimelyFreeze pipeline step on the local GPU."""

    def __init__(self, shape: ModelShape, schedule: str = "gpipe", ranks: int = 1, stages_per_rank: int = 1,
                 microbatches: int = 8, rank: int = 0, phases=(2, 8, 10, 20), r_max: float = 0.8, lr: float = 1e-3,
                 seed: int = 42, apf: bool = False, apf_alpha: float = 0.9, apf_threshold: float = 1e-4,
                 apf_every: int = 1, device: int = 0, mask_threads: int = 0, hybrid: bool = False,
                 hybrid_unit_fraction: float = 0.5, optimizer: str = "sgd", betas=(0.9, 0.999), eps: float = 1e-8,
                 weight_decay: float = 0.0):
        self.lib = _native.device()
        self.shape = shape
        self.M = microbatches
        self.S = ranks * stages_per_rank
        m = PfModelCfg(shape.hidden, shape.ffn, shape.n_heads, shape.n_kv_heads, shape.head_dim, shape.vocab,
                       shape.layers, shape.seq, shape.micro_batch, shape.rope_theta, shape.norm_eps, shape.init_std,
                       shape.family, shape.image, shape.patch, shape.channels)
        c = PfTrainCfg()
        c.kind = KINDS[schedule]
        self.kinds = 3 if c.kind in SPLIT_KINDS else 2  # action kinds per cell: f, b (, w)
        c.ranks, c.stages_per_rank, c.microbatches, c.rank = ranks, stages_per_rank, microbatches, rank
        c.phases[:] = list(phases)
        c.r_max, c.lr, c.seed = r_max, lr, seed
        c.apf, c.apf_every, c.apf_alpha, c.apf_threshold = int(apf), apf_every, apf_alpha, apf_threshold
        c.device, c.mask_threads = device, mask_threads
        c.hybrid, c.hybrid_unit_fraction = int(hybrid), hybrid_unit_fraction
        if optimizer not in ("sgd", "adamw"):
            raise ValueError(f"optimizer must be 'sgd' or 'adamw', got {optimizer!r}")
        c.optimizer = 1 if optimizer == "adamw" else 0
        c.beta1, c.beta2, c.eps, c.weight_decay = betas[0], betas[1], eps, weight_decay
        self.phases = tuple(phases)
        self._ctx = ctypes.c_void_p()
        _check(self.lib.pf_trainer_create(ctypes.byref(m), ctypes.byref(c), ctypes.byref(self._ctx)), "trainer_create")
        self.info = self.get_info()

    def init_comm(self) -> None:
        """Set up the NCCL P2P transport for a multi-rank pipeline (call on every rank).

        Rank 0 creates the ncclUniqueIds (the world communicator, then one two-rank
        communicator per P2P link, see links()) and shares them over the default
        torch.distributed group."""
        import torch.distributed as dist

        world, rank = dist.get_world_size(), dist.get_rank()
        n = ctypes.c_int(0)
        _check(self.lib.pf_trainer_comm_ids(self._ctx, ctypes.byref(n)), "comm_ids")
        obj = [None]
        if rank == 0:
            buf = ctypes.create_string_buffer(n.value * 128)
            _check(self.lib.pf_nccl_unique_ids(buf, n.value), "nccl_unique_ids")
            obj = [bytes(buf.raw)]
        dist.broadcast_object_list(obj, src=0)
        ids = ctypes.create_string_buffer(obj[0], n.value * 128)
        _check(self.lib.pf_trainer_init_comm(self._ctx, ids, world, rank), "trainer_init_comm")

    def links(self) -> list[tuple[int, int, int]]:
        """P2P links of the pipeline: (kind 0 activations / 1 gradients, src rank, dst rank)."""
        n = ctypes.c_int(0)
        _check(self.lib.pf_trainer_comm_ids(self._ctx, ctypes.byref(n)), "comm_ids")
        out = np.zeros(max(1, 3 * (n.value - 1)), dtype=np.int32)
        _check(self.lib.pf_trainer_links(self._ctx, out.ctypes.data_as(ctypes.c_void_p)), "links")
        return [tuple(int(x) for x in out[3 * k:3 * k + 3]) for k in range(n.value - 1)]

    def close(self) -> None:
        if self._ctx:
            self.lib.pf_trainer_destroy(self._ctx)
            self._ctx = ctypes.c_void_p()

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    def _host_ids(self, a: np.ndarray | None, what: str):
        """[M, T] int32 C-contiguous (the C side copies M*T*4 bytes); keeps the array alive."""
        if a is None:
            return None, None
        if not (isinstance(a, np.ndarray) and a.dtype == np.int32 and a.flags.c_contiguous):
            a = np.ascontiguousarray(a, dtype=np.int32)
        if a.size != self.M * self.shape.tokens:
            raise ValueError(f"{what}: need {self.M} x {self.shape.tokens} ids, got shape {a.shape}")
        return a, a.ctypes.data_as(ctypes.c_void_p)

    def step(self, t: int, tokens: np.ndarray | None = None, targets: np.ndarray | None = None,
             masks: np.ndarray | None = None) -> dict:
        """One training step. masks: caller-owned frozen-unit masks of every local cell (per local
        stage, M masks of ceil(units/64) uint64 words, FreezeMask::test bit order) instead of the
        controller's (pf_trainer_step_masks)."""
        r = PfStepResult()
        tokens, tp = self._host_ids(tokens, "tokens")
        targets, gp = self._host_ids(targets, "targets")
        if masks is None:
            _check(self.lib.pf_trainer_step(self._ctx, t, tp, gp, ctypes.byref(r)), f"trainer_step(t={t})")
        else:
            need = sum(self.M * ((self.stage_buffers(i)["n_units"] + 63) // 64) for i in range(self.info["local_stages"]))
            mk = np.ascontiguousarray(masks, dtype=np.uint64)
            if mk.size != need:
                raise ValueError(f"masks: need {need} words, got {mk.size}")
            _check(self.lib.pf_trainer_step_masks(self._ctx, t, tp, gp, mk.ctypes.data_as(ctypes.c_void_p),
                                                  ctypes.byref(r)), f"trainer_step_masks(t={t})")
        return {k: getattr(r, k) for k, _ in PfStepResult._fields_}

    def set_override(self, ratio: float | None) -> None:
        _check(self.lib.pf_trainer_set_override(self._ctx, -1.0 if ratio is None else float(ratio)), "set_override")

    def set_plan(self, ratios) -> None:
        r = np.ascontiguousarray(ratios, dtype=np.float64)
        _check(self.lib.pf_trainer_set_plan(self._ctx, r.ctypes.data_as(ctypes.c_void_p)), "set_plan")

    def get_plan(self):
        ratios = np.zeros(self.S * self.M)
        out3 = np.zeros(3)
        wmin = np.zeros(self.kinds * self.S * self.M)
        wmax = np.zeros(self.kinds * self.S * self.M)
        rc = self.lib.pf_trainer_get_plan(self._ctx, *(a.ctypes.data_as(ctypes.c_void_p) for a in (ratios, out3, wmin, wmax)))
        if rc == _native.PF_ERR_DOMAIN:
            return None
        _check(rc, "get_plan")
        return dict(ratios=ratios, makespan_base=out3[0], makespan_opt=out3[1], makespan_floor=out3[2],
                    w_min=wmin, w_max=wmax)

    def action_ms(self):
        n = self.info["actions"]
        ms = np.zeros(n)
        kinds = np.zeros(n, dtype=np.int32)
        mbs = np.zeros(n, dtype=np.int32)
        st = np.zeros(n, dtype=np.int32)
        _check(self.lib.pf_trainer_action_ms(self._ctx, *(a.ctypes.data_as(ctypes.c_void_p) for a in (ms, kinds, mbs, st))),
               "action_ms")
        return ms, kinds, mbs, st

    def action_times(self):
        """(start_ms, end_ms, kinds, microbatches, stages) of the last step's actions on this rank."""
        ms, kinds, mbs, st = self.action_ms()
        start = np.zeros(len(ms))
        _check(self.lib.pf_trainer_action_starts(self._ctx, start.ctypes.data_as(ctypes.c_void_p)), "action_starts")
        return start, start + ms, kinds, mbs, st

    def get_info(self) -> dict:
        i = PfTrainerInfo()
        _check(self.lib.pf_trainer_get_info(self._ctx, ctypes.byref(i)), "get_info")
        return {k: getattr(i, k) for k, _ in PfTrainerInfo._fields_}

    def stage_buffers(self, local_stage: int = 0) -> dict:
        ptrs = [ctypes.c_void_p() for _ in range(4)]
        n = ctypes.c_longlong()
        u = ctypes.c_int()
        _check(self.lib.pf_trainer_stage_buffers(self._ctx, local_stage, *(ctypes.byref(p) for p in ptrs),
                                                 ctypes.byref(n), ctypes.byref(u)), "stage_buffers")
        return dict(master=ptrs[0].value, weights=ptrs[1].value, grad=ptrs[2].value, stamps=ptrs[3].value,
                    n_params=n.value, n_units=u.value)

    def optim_state(self, local_stage: int = 0) -> dict:
        """AdamW state pointers of a local stage (None before the first AdamW step)."""
        ptrs = [ctypes.c_void_p() for _ in range(3)]
        _check(self.lib.pf_trainer_optim_state(self._ctx, local_stage, *(ctypes.byref(p) for p in ptrs)),
               "optim_state")
        return dict(m=ptrs[0].value, v=ptrs[1].value, unit_steps=ptrs[2].value)

    def apf_base(self, local_stage: int = 0):
        """Hybrid mode: APF base unit set of the last APF step (None before the first one)."""
        units = self.stage_buffers(local_stage)["n_units"]
        out = np.zeros(max(1, (units + 63) // 64), dtype=np.uint64)
        rc = self.lib.pf_trainer_apf_base(self._ctx, local_stage, out.ctypes.data_as(ctypes.c_void_p))
        if rc == _native.PF_ERR_DOMAIN:
            return None
        _check(rc, "apf_base")
        return out[: (units + 63) // 64]

    def last_masks(self, local_stage: int = 0) -> np.ndarray:
        units = self.stage_buffers(local_stage)["n_units"]
        words = (units + 63) // 64
        out = np.zeros((self.M, words), dtype=np.uint64)
        _check(self.lib.pf_trainer_last_masks(self._ctx, local_stage, out.ctypes.data_as(ctypes.c_void_p)), "last_masks")
        return out


def shape_dict(shape: ModelShape) -> dict:
    return asdict(shape)
