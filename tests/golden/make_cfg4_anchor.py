"""Full-size cfg4 (729^3) oracle anchor: the first CG iterations of the CPU oracle.

SURVEY 8(c) item 2: a full-size oracle solve of cfg4 is infeasible, but a few
iterations fit a host with >= ~200 GB (the GPU box has 196 GB and 16 cores), so
``max_iter = 3`` of the memory-lean oracle restatement (``oracle/lean_cg.py``,
pinned against the reference's goldens) pins the 729^3 device solve.

Run ON THE GPU BOX (the device generator builds the Voronoi labels; the host
generator ``generators.voronoi_labels`` is bit-identical to it but takes hours
at 729^3 -- ``tests/test_gpu_parity.py`` checks that identity at 81^3):

    python tests/golden/make_cfg4_anchor.py labels /tmp/cfg4_labels.npy
    (ulimit -v 170000000; python tests/golden/make_cfg4_anchor.py solve /tmp/cfg4_labels.npy \
        gpurun_out/cfg4_729_anchor.npz)

(two processes: the oracle runs without a CUDA context, under an address-space
limit, so a memory overrun fails with MemoryError instead of taking the host down)

then copy the file to ``tests/golden/``.  Stored: iterations, the residual
history r_0..r_3, |x|, the energy <A(E + x), E + x> and x at 4096 seeded
sample positions of the (3, 729, 729, 729) solution.
"""

from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

N = 729
MAX_ITER = 3
SAMPLE_SEED = 424242
NSAMPLE = 4096
E = (1.0, 0.0, 0.0)


def sample_idx(n):
    return np.sort(np.random.default_rng(SAMPLE_SEED).choice(n, size=min(NSAMPLE, n), replace=False))


def device_labels(n):
    from paper_1311_0089_b200 import _native, generators as gen
    from paper_1311_0089_b200.grid import GridSpec

    seeds, packed = gen.cfg4_grains(512, gen.SEEDS["cfg4"], n)
    ctx = _native.Context(GridSpec((1.0,) * 3, (n,) * 3), 0)
    labels = ctx.generate_voronoi(seeds, packed, want_labels=True)
    del ctx
    return labels.reshape(n, n, n), packed


def make_labels(path):
    labels, _ = device_labels(N)
    np.save(path, labels)


def main(labels_path, out):
    from oracle import lean_cg
    from paper_1311_0089_b200 import generators as gen

    t0 = time.time()
    labels = np.load(labels_path)
    _, grains = gen.cfg4_grains(512, gen.SEEDS["cfg4"], N)
    field = np.empty((6, N, N, N))
    for m in range(6):
        np.take(grains[:, m], labels, out=field[m])
    del labels
    print(f"field built {time.time() - t0:.1f} s", flush=True)
    op = lean_cg.LeanOperator((N,) * 3, (1.0,) * 3, packed=field)
    rep = lean_cg.solve_cg(op, E, 1e-8, MAX_ITER,
                           on_iter=lambda i, h: print(f"iter {i} |r| {h:.17e} {time.time() - t0:.1f} s", flush=True))
    x = rep["solution"]
    idx = sample_idx(x.size)
    # energy <A (E + x), E + x> (homogenize.py:59-67)
    for a in range(3):
        x[a] += E[a]
    flux = np.empty_like(x)
    op.apply_A(x, flux)
    energy = op.inner(flux, x)
    del flux
    for a in range(3):
        x[a] -= E[a]
    np.savez_compressed(out, iterations=rep["iterations"], history=np.array(rep["history"]),
                        norm=float(np.sqrt(op.inner(x, x))), energy=energy, sample_idx=idx,
                        sample=x.reshape(-1)[idx], max_iter=MAX_ITER, n=N,
                        seconds=time.time() - t0)
    print(f"wrote {out}: history {rep['history']} energy {energy!r} ({time.time() - t0:.1f} s)", flush=True)


if __name__ == "__main__":
    if sys.argv[1] == "labels":
        make_labels(sys.argv[2])
    else:
        main(sys.argv[2], sys.argv[3])
