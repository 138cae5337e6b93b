"""Times the one-call decompose_quantize / dequantize_recompose against the
two-call sequences on the 513^3 fp32 bench field (CUDA events, synchronous
calls: the quantizer returns its outlier count)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2010_05872_b200 as mg
import synthetic_fields as sf


def timeit(fn, n=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 513
    d = sf.config2_field((n, n, n), seed=0, device="cuda").contiguous()
    h = mg.GridHierarchy.create(tuple(d.shape))
    ws = mg.SolverWorkspace()
    r = float(d.max() - d.min())
    for rel in (1e-2, 1e-3, 1e-4):
        plan = mg.make_plan(mg.QuantMode.levelwise, rel * r / 4, h)
        mc = mg.decompose(d, h, 0, ws)
        s = mg.quantize(mc, plan, ws)
        t_dec = timeit(lambda: mg.decompose(d, h, 0, ws))
        t_q = timeit(lambda: mg.quantize(mc, plan, ws))
        t_two = timeit(lambda: mg.quantize(mg.decompose(d, h, 0, ws), plan, ws))
        t_one = timeit(lambda: mg.decompose_quantize(d, h, plan, 0, ws))
        t_rec = timeit(lambda: mg.recompose(mc, ws))
        t_dq = timeit(lambda: mg.dequantize(s, plan, h, ws))
        t_two_r = timeit(lambda: mg.recompose(mg.dequantize(s, plan, h, ws), ws))
        t_one_r = timeit(lambda: mg.dequantize_recompose(s, plan, h, ws))
        print(f"rel {rel:g}: outliers {s.outlier_positions.numel()}  decompose {t_dec:.3f} quantize {t_q:.3f} "
              f"two calls {t_two:.3f} one call {t_one:.3f} ms | recompose {t_rec:.3f} dequantize {t_dq:.3f} "
              f"two calls {t_two_r:.3f} one call {t_one_r:.3f} ms", flush=True)


if __name__ == "__main__":
    main()
