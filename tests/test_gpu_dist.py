"""One process per GPU over NCCL (fc_create_dist), two real ranks (needs >= 2 GPUs;
skipped otherwise -- NCCL rejects two ranks on one device, and the slab logic is
covered on one GPU by tests/test_gpu_sharded.py).

Each rank owns one axis-0 slab.  Both exchange transports run: the fused one
(default: the forward middle sweep and the outer sweep store straight into the
peer process's spectrum buffers, mapped with CUDA IPC; NCCL only orders the
phases) and the NCCL send / receive copies (plan option fused_exchange = 0).
They perform the same arithmetic, so their CG / fixed-point solutions must be
bitwise identical; both must match the single-GPU solve to rounding with
identical iteration counts."""

import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]

WORKER = r'''
import json, os, sys
import numpy as np
sys.path.insert(0, ROOT)
import torch.distributed as dist
from paper_1311_0089_b200 import _native, generators as gen, parallel
from paper_1311_0089_b200.grid import GridSpec

dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
out = {}
for name, n in (("cfg3", 81), ("cfg5", 45)):
    a = gen.cfg3_sphere(n) if name == "cfg3" else gen.cfg5_two_phase(n)
    E = np.array([[1.0, 0.0, 0.0], [0.3, -0.2, 1.0]])
    res = {}
    for fused in (1, 0):
        with _native.plan_options(fused_exchange=fused):
            ctx = parallel.distributed_context(a.spec, device=rank)
        ctx.set_coefficients(a)
        reps, x, _ = ctx.solve_cg(E, 1e-8, 1000)
        freps, fx = ctx.solve_fixed_point(E[:1], 1e-6, 2000, 25.5 * np.eye(3), np.ones(1))
        xg = parallel.gather_slabs(x, 2, world, rank)
        fg = parallel.gather_slabs(fx, 2, world, rank)
        res[fused] = ([r["iterations"] for r in reps], xg, freps[0]["iterations"], fg)
        del ctx
    if rank == 0:
        one = _native.Context(a.spec, 0)
        one.set_coefficients(a)
        r1, x1, _ = one.solve_cg(E, 1e-8, 1000)
        f1, fx1 = one.solve_fixed_point(E[:1], 1e-6, 2000, 25.5 * np.eye(3), np.ones(1))
        out[name] = {
            "its_fused": res[1][0], "its_copy": res[0][0], "its_one": [r["iterations"] for r in r1],
            "fused_eq_copy": bool(np.array_equal(res[1][1], res[0][1])),
            "fp_fused_eq_copy": bool(np.array_equal(res[1][3], res[0][3])),
            "rel_vs_one": float(np.linalg.norm(res[1][1] - x1) / np.linalg.norm(x1)),
            "fp_its": [res[1][2], res[0][2], f1[0]["iterations"]],
            "fp_rel_vs_one": float(np.linalg.norm(res[1][3] - fx1) / np.linalg.norm(fx1)),
        }
if rank == 0:
    json.dump(out, open(OUT, "w"))
dist.destroy_process_group()
'''


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_two_ranks_fused_and_nccl_exchanges(tmp_path):
    from paper_1311_0089_b200 import _native

    if _native.device_count() < 2:
        pytest.skip("needs >= 2 GPUs (NCCL rejects two ranks on one device)")
    script = tmp_path / "worker.py"
    out = tmp_path / "out.json"
    script.write_text(f"ROOT = {str(ROOT)!r}\nOUT = {str(out)!r}\n" + WORKER)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), str(script)]
    proc = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=dict(os.environ))
    assert proc.returncode == 0, proc.stderr[-3000:]
    res = json.loads(out.read_text())
    for name, r in res.items():
        assert r["its_fused"] == r["its_copy"] == r["its_one"], (name, r)
        assert r["fused_eq_copy"] and r["fp_fused_eq_copy"], (name, r)
        assert r["rel_vs_one"] <= 1e-12 and r["fp_rel_vs_one"] <= 1e-12, (name, r)
        assert r["fp_its"][0] == r["fp_its"][1] == r["fp_its"][2], (name, r)
