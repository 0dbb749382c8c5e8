"""Host-side tests of the C-ABI library (no GPU needed): it builds, loads,
exports every symbol include/sttsv.h declares, validates inputs before any
device work, and shards edges as documented."""
import os
import re
import subprocess

import numpy as np
import pytest

import paper_2311_08595_b200 as S
import workloads as W

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "sttsv.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sttsv_[a-z_]+)\s*\(", src)))


def test_exports_every_declared_symbol():
    lib = S.load()
    decl = declared_symbols()
    assert len(decl) >= 14
    for name in decl:
        assert hasattr(lib, name), name
    assert set(decl) == set(S.exported_symbols())
    assert "sm_100a" in S.sttsv_version()


def test_status_strings():
    for code, name in S.sttsv.STATUS.items():
        assert S.sttsv_status_string(code) == name


@pytest.mark.parametrize("sizes,idx,w,N,n,flags,err", [
    ([2], [3, 1], None, 4, 10, 0, "STTSV_ERR_UNSORTED"),
    ([2], [3, 3], None, 4, 10, 0, "STTSV_ERR_REPEATED_VERTEX"),
    ([2], [3, 3], None, 4, 10, 1, "STTSV_ERR_REPEATED_VERTEX"),
    ([2], [3, 10], None, 4, 10, 0, "STTSV_ERR_VERTEX_RANGE"),
    ([2], [-1, 3], None, 4, 10, 0, "STTSV_ERR_VERTEX_RANGE"),
    ([5], [0, 1, 2, 3, 4], None, 4, 10, 0, "STTSV_ERR_EDGE_SIZE"),
    ([0], [], None, 4, 10, 0, "STTSV_ERR_EDGE_SIZE"),
    ([2], [1, 3], [float("nan")], 4, 10, 0, "STTSV_ERR_NONFINITE"),
    ([2], [1, 3], [float("inf")], 4, 10, 0, "STTSV_ERR_NONFINITE"),
    ([2], [1, 3], None, 0, 10, 0, "STTSV_ERR_INVALID_ARGUMENT"),
    ([2], [1, 3], None, 33, 10, 0, "STTSV_ERR_INVALID_ARGUMENT"),
    ([2], [1, 3], None, 4, 0, 0, "STTSV_ERR_INVALID_ARGUMENT"),
    ([2], [1, 3], None, 4, 10, 1 << 5, "STTSV_ERR_UNSUPPORTED"),
])
def test_validation_errors(sizes, idx, w, N, n, flags, err):
    with pytest.raises(S.SttsvError) as ei:
        S.sttsv_plan_create(n, N, np.array(sizes, np.int32), np.array(idx, np.int32),
                            None if w is None else np.array(w), flags=flags)
    assert ei.value.name == err
    assert S.sttsv_last_error()


def test_bad_world_rank():
    for world, rank in ((0, 0), (2, 2), (2, -1)):
        with pytest.raises(S.SttsvError) as ei:
            S.sttsv_plan_create(10, 3, np.array([2], np.int32), np.array([1, 2], np.int32), world=world, rank=rank)
        assert ei.value.name == "STTSV_ERR_INVALID_ARGUMENT"


def test_shard_edges_partition():
    hg = W.generate("mid", m=10_001, n=5_000)
    for world in (1, 2, 3, 8):
        parts = [S.sttsv_shard_edges(hg.sizes, hg.rank, world, r) for r in range(world)]
        allp = np.concatenate(parts)
        assert len(allp) == hg.m and len(np.unique(allp)) == hg.m
        # every bucket is split into contiguous, balanced, input-ordered slices
        for k in range(1, hg.rank + 1):
            per = [p[hg.sizes[p] == k] for p in parts]
            cnt = [len(q) for q in per]
            assert max(cnt) - min(cnt) <= 1
            cat = np.concatenate(per)
            assert np.all(np.diff(cat) > 0)
            assert np.array_equal(cat, np.where(hg.sizes == k)[0])


def _build_c_client(tmp_path):
    lib = S.load()._name
    exe = tmp_path / "abi_c11"
    subprocess.check_call(["gcc", "-std=c11", "-Wall", "-Wextra", "-Werror", "-pedantic",
                           "-I", os.path.join(ROOT, "include"), os.path.join(ROOT, "tests", "c", "abi_c11.c"),
                           lib, "-Wl,-rpath," + os.path.dirname(lib), "-lm", "-o", str(exe)])
    return exe


def test_plain_c_client_host(tmp_path):
    """include/sttsv.h compiles as C11 (gcc -std=c11 -pedantic -Werror) and links against
    libsttsv.so; the host-only calls behave as documented."""
    exe = _build_c_client(tmp_path)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "abi_c11 ok" in out.stdout


@pytest.mark.gpu
def test_plain_c_client_fig1(tmp_path):
    """The C client drives plan_create -> apply_host -> destroy on Fig. 1
    and gets the degree vector (3,2,3,4,2,3,3,1)."""
    exe = _build_c_client(tmp_path)
    out = subprocess.run([str(exe), "gpu"], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "fig1 y = (3,2,3,4,2,3,3,1)" in out.stdout
