"""HBM throughput of the freeze-side kernels at the LLaMA-1B stage size (16 layers + LM head,
1.23 B freezable parameters in 75,424 128x128 units), CUDA events, one B200:

  K6      masked SGD over the touched units (theta -= scale G, bf16 copy):   14 B / touched param
  K6+K4   the same with the APF EMA update fused (every unit's E, E_abs):    + 16 B / unit param
  K4      standalone apf_update (delta in, E, E_abs, score):                 24 B / param

Touched = units unfrozen in at least one of the step's 8 microbatches at the LP-stable ratio
0.8 (1 - 0.8^8 = 83%). Prints one line per kernel: time, algorithmic GB/s, fraction of the
measured HBM peak (MEASURED_PEAKS.json).
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2602_05754_b200 import _native  # noqa: E402

lib = _native.device()


def unit_table(shapes):
    dt = np.dtype([("elem_offset", "<i8"), ("rows", "<i4"), ("cols", "<i4"), ("unit_offset", "<i4"),
                   ("tiles_n", "<i4"), ("units", "<i4"), ("pair_offset", "<i4")])
    tab = np.zeros(len(shapes), dtype=dt)
    off = u = 0
    for i, (r, c) in enumerate(shapes):
        tn, tm = (c + 127) // 128, (r + 127) // 128
        tab[i] = (off, r, c, u, tn, tm * tn, 0)
        off = (off + r * c + 63) // 64 * 64
        u += tm * tn
    return tab, off, u


def timed(fn, iters=10):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def main():
    peak = 6545.3
    try:
        peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    except (OSError, KeyError, ValueError):
        pass
    shapes = [(3072, 2048), (2048, 2048), (16384, 2048), (2048, 8192)] * 16 + [(128256, 2048)]
    tab, n, U = unit_table(shapes)
    rng = np.random.default_rng(0)
    touched_units = rng.random(U) < 1.0 - 0.8 ** 8
    st = torch.tensor(np.where(touched_units, 7, 0).astype(np.int32), device="cuda")
    per_unit = np.zeros(U, dtype=np.int64)
    for e in tab:
        tn = int(e["tiles_n"])
        for lu in range(int(e["units"])):
            rb, cb = divmod(lu, tn)
            per_unit[int(e["unit_offset"]) + lu] = (min(128, int(e["rows"]) - rb * 128) *
                                                    min(128, int(e["cols"]) - cb * 128))
    unit_params = int(per_unit.sum())
    touched_params = int(per_unit[touched_units].sum())
    master = torch.zeros(n, device="cuda")
    weights = torch.zeros(n, dtype=torch.bfloat16, device="cuda")
    grad = torch.randn(n, device="cuda")
    ema = torch.zeros(n, device="cuda")
    ema_abs = torch.zeros(n, device="cuda")
    score = torch.zeros(n, device="cuda")
    elig = torch.zeros(U, dtype=torch.int32, device="cuda")
    td = torch.tensor(tab.view(np.uint8), device="cuda")
    s = torch.cuda.current_stream().cuda_stream

    def k6():
        assert lib.pf_masked_sgd_units(master.data_ptr(), weights.data_ptr(), grad.data_ptr(), st.data_ptr(), 7, 1e-4,
                                       td.data_ptr(), len(tab), U, None, None, 0.0, 0.0, None, s) == 0

    def k6_apf():
        assert lib.pf_masked_sgd_units(master.data_ptr(), weights.data_ptr(), grad.data_ptr(), st.data_ptr(), 7, 1e-4,
                                       td.data_ptr(), len(tab), U, ema.data_ptr(), ema_abs.data_ptr(), 0.9, 1e-4,
                                       elig.data_ptr(), s) == 0

    def k4():
        assert lib.pf_apf_update(ema.data_ptr(), ema_abs.data_ptr(), grad.data_ptr(), score.data_ptr(), unit_params,
                                 0.9, s) == 0

    print(f"stage: {U} units, {unit_params / 1e9:.3f} B unit params, {touched_params / 1e9:.3f} B touched "
          f"({touched_units.mean():.3f} of units); HBM peak {peak} GB/s (measured)")
    for name, fn, nbytes in [("K6 masked SGD", k6, 14 * touched_params),
                             ("K6 masked SGD + fused K4 APF", k6_apf, 14 * touched_params + 16 * unit_params),
                             ("K4 apf_update standalone", k4, 24 * unit_params)]:
        ms = timed(fn)
        gbs = nbytes / (ms * 1e-3) / 1e9
        print(f"{name:30s} {ms:7.3f} ms  {nbytes / 1e9:6.2f} GB algorithmic  {gbs:7.0f} GB/s  {gbs / peak:.3f} of peak",
              flush=True)


if __name__ == "__main__":
    main()
