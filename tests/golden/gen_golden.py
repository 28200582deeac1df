"""Generate the golden vectors in tests/golden/ from the REFERENCE ITSELF.

Runs the reference's own C++ sources (compiled unmodified by oracle/Makefile into
oracle/_ref/libdfx_ref.so, namespace renamed) on inputs drawn with the reference's own
fixtures (seeded_fixture / gaussian_fixture / gaussian_vector / derive_seed), and stores
inputs + outputs as .npz.  /root/reference does not exist on the GPU box, so these
fixtures are what pins GPU parity there.  Re-run here with:

    make -C oracle && python tests/golden/gen_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
import pyoracle  # noqa: E402


def kappa(W, A, B, s):
    BA = B.astype(np.float64) @ A.astype(np.float64)
    W64 = W.astype(np.float64)
    base, cross, ba = (W64 * W64).sum(1), (W64 * BA).sum(1), (BA * BA).sum(1)
    n2 = base + 2 * s * cross + s * s * ba
    return (base + np.abs(2 * s * cross) + s * s * ba) / np.maximum(n2, 1e-300)


def gen_compose(R):
    out = {}
    k = 0
    # test_compose.cpp:94-114 inputs (60 ragged trials), every third one
    for trial in range(0, 60, 3):
        seed = R.derive_seed(12345, trial)
        rows, d_out = 1 + seed % 70, 1 + R.derive_seed(seed, 1) % 200
        dt = trial % 3
        s = 0.0 if trial % 7 == 0 else 0.9
        base = R.gaussian_fixture(rows, d_out, 0.0, 3.0, R.derive_seed(seed, 2), dt)
        lora = R.gaussian_fixture(rows, d_out, 0.0, 3.0, R.derive_seed(seed, 3), dt)
        g = np.array([R.round_to_dtype(v, dt) for v in R.gaussian_vector(d_out, 1.0, 0.05,
                                                                          R.derive_seed(seed, 4))])
        delta, inner = R.compose(2, dt, base, lora, g, s, need_inner=True)
        stable, _ = R.compose(0, dt, base, lora, g, s)
        assert np.array_equal(stable.view(np.uint32), delta.view(np.uint32))
        out.update({f"c{k}_dt": dt, f"c{k}_s": s, f"c{k}_base": base, f"c{k}_lora": lora,
                    f"c{k}_g": g.astype(np.float32), f"c{k}_delta": delta, f"c{k}_inner": inner})
        k += 1
    # an aligned block that exercises the vectorised kernels
    for dt in (0, 1, 2):
        base = R.gaussian_fixture(64, 512, 0.0, 4.0, 900 + dt, dt)
        lora = R.gaussian_fixture(64, 512, 0.0, 4.0, 910 + dt, dt)
        g = np.array([R.round_to_dtype(v, dt) for v in R.gaussian_vector(512, 1.0, 0.002, 920 + dt)])
        delta, inner = R.compose(2, dt, base, lora, g, 0.1020620726159658, need_inner=True)
        out.update({f"c{k}_dt": dt, f"c{k}_s": 0.1020620726159658, f"c{k}_base": base,
                    f"c{k}_lora": lora, f"c{k}_g": g.astype(np.float32), f"c{k}_delta": delta,
                    f"c{k}_inner": inner})
        k += 1
    out["n_cases"] = k
    b = 0
    for rows, d_out, dt in [(6, 10, 0), (33, 129, 1), (100, 64, 2), (256, 512, 1), (77, 96, 0)]:
        dy = R.gaussian_fixture(rows, d_out, 0.0, 1.0, 51 + b, dt)
        inner = R.gaussian_fixture(rows, d_out, 0.0, 1.0, 61 + b, dt)
        g = np.array([R.round_to_dtype(v, dt) for v in R.gaussian_vector(d_out, 1.0, 0.05, 71 + b)])
        wn = np.array([R.round_to_dtype(2.0 + 0.37 * j, dt) for j in range(d_out)])
        dl, db, dm = R.compose_bwd(dt, dy, g, 0.8, inner, wn, mag_grad=True)
        out.update({f"b{b}_dt": dt, f"b{b}_s": 0.8, f"b{b}_dy": dy, f"b{b}_inner": inner,
                    f"b{b}_g": g.astype(np.float32), f"b{b}_wn": wn.astype(np.float32),
                    f"b{b}_dlora": dl, f"b{b}_dbase": db, f"b{b}_dmag": dm.astype(np.float32)})
        b += 1
    out["n_bwd"] = b
    return out


def gen_norm(R):
    out = {}
    k = 0
    cases = []
    # test_factored_norm.cpp:62-76 shape grid (fp32)
    seed = 4000
    dims, ranks = [3, 17, 64, 96, 257], [1, 2, 8, 33]
    for d_out in dims:
        for d_in in dims:
            r = ranks[(d_out + d_in) % 4]
            s = 1.0 if d_out % 2 else 2.0 / np.sqrt(r)
            seed += 1
            cases.append((0, d_out, d_in, r, s, seed))
            seed += 1
    # bf16 cases, incl. shapes on the tensor-core path
    cases += [(1, 64, 96, 8, 1.0, 200), (1, 256, 512, 64, 0.25, 210), (1, 384, 1024, 128, 0.2, 220),
              (2, 64, 96, 8, 1.0, 230), (0, 32, 257, 4, 0.7, 300), (0, 16, 48, 5, 0.0, 400)]
    for dt, d_out, d_in, r, s, sd in cases:
        W = R.seeded_gaussian(d_out, d_in, R.derive_seed(sd, 0), dt)
        A = R.seeded_gaussian(r, d_in, R.derive_seed(sd, 1), dt)
        B = R.seeded_gaussian(d_out, r, R.derive_seed(sd, 2), dt)
        cs, _ = R.plan_chunks(d_out, d_in)
        base, cross, ba = R.norm_terms(dt, W, A, B, s, cs)
        norm = R.row_norm(dt, W, A, B, s, cs)
        f64 = R.dense_row_norm_f64(W, A, B, s)
        out.update({f"n{k}_dt": dt, f"n{k}_s": s, f"n{k}_cs": cs, f"n{k}_W": W, f"n{k}_A": A,
                    f"n{k}_B": B, f"n{k}_base": base, f"n{k}_cross": cross, f"n{k}_ba": ba,
                    f"n{k}_norm": norm.astype(np.float32), f"n{k}_f64": f64,
                    f"n{k}_kappa": kappa(W, A, B, s)})
        k += 1
    out["n_cases"] = k
    # assemble / magnitude known answers (test_factored_norm.cpp:142-192)
    return out


def main():
    R = pyoracle.Reference()
    np.savez_compressed(os.path.join(HERE, "compose.npz"), **gen_compose(R))
    np.savez_compressed(os.path.join(HERE, "norm.npz"), **gen_norm(R))
    for f in ("compose.npz", "norm.npz"):
        print(f, os.path.getsize(os.path.join(HERE, f)), "bytes")


if __name__ == "__main__":
    main()
