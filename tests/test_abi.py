"""CPU checks of the boundary: the C-ABI library builds, loads and exports every
symbol include/eucalc.h declares (no compute calls without a GPU); host-side
logic of the binding."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "eucalc.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(eucalc_[a-z_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("eucalc_build_complex", "eucalc_critical_points", "eucalc_ect", "eucalc_radon", "eucalc_hybrid"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    from paper_2405_02256_b200 import _build

    _build.build()
    lib = ctypes.CDLL(_build.LIB)
    for s in declared_symbols():
        assert hasattr(lib, s), s


def test_status_strings_without_gpu():
    import paper_2405_02256_b200 as eu

    L = eu.lib()
    assert L.eucalc_status_string(0) == b"ok"
    assert L.eucalc_status_string(eu.E_NONGENERIC).startswith(b"non-generic")


def test_native_code_targets_sm100a():
    """The library carries sm_100a SASS (cuobjdump), not PTX-only or another arch."""
    import subprocess

    from paper_2405_02256_b200 import _build

    _build.build()
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _build.LIB], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_no_oracle_import_in_product():
    """The product package never imports the oracle (independence)."""
    pkg = os.path.join(ROOT, "paper_2405_02256_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dp, f)).read()
                assert "import oracle" not in txt and "eucalc_oracle" not in txt, f


def test_gloo_world2_direction_sharding():
    """Multi-process host logic (gloo, world_size 2): the weak-scaling shard of
    (image, direction) work units used by bench.py --gpus N covers every unit once."""
    import torch.multiprocessing as mp

    mp.start_processes(_shard_worker, args=(2,), nprocs=2, join=True, start_method="spawn")


def _shard_worker(rank, world):
    import os

    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ.setdefault("MASTER_PORT", "29533")
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench

    nimg = 37
    mine = bench.shard_range(nimg, rank, world)
    t = torch.zeros(nimg, dtype=torch.int64)
    t[mine[0]:mine[1]] += 1
    dist.all_reduce(t)
    assert bool((t == 1).all())
    # single-image configs: directions split by orthant pair into contiguous chunks
    import numpy as np

    import paper_2405_02256_b200 as eu
    import synth

    dirs = synth.random_directions(101, 3, 8, 5)
    idx, sub = eu.shard_directions(dirs, rank, world)
    assert np.array_equal(sub, dirs[idx])
    u = torch.zeros(len(dirs), dtype=torch.int64)
    u[torch.from_numpy(idx)] += 1
    dist.all_reduce(u)
    assert bool((u == 1).all())
    e = ((sub > 0).astype(np.int64) << np.arange(3)).sum(1)
    pair = np.where((e >> 2) & 1, e ^ 7, e)
    assert np.all(np.diff(pair) >= 0)  # one orthant pair's directions stay together on a rank
    dist.destroy_process_group()


def test_bench_entry_gloo_world2():
    """bench.py's own multi-GPU entry (--gpus 2 re-launches itself under
    torch.distributed.run) on CPU with gloo: two ranks rendezvous on 127.0.0.1,
    each takes its shard, the time is the max over ranks and rank 0 alone prints
    one JSON line with n_gpus = 2."""
    import json
    import sys

    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--plumbing-check",
                          "--steps", "2", "--warmup", "3"], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["plumbing_check"] and line["value"] > 0
    shards = sorted(tuple(s) for s in line["shards"])
    assert [s[0] for s in shards] == [0, 1] and shards[0][2] == shards[1][1] and shards[1][2] == 1024
    assert shards[0][3] != shards[1][3]  # each rank draws its own images (weak scaling)
