"""Host-side checks of the C ABI (no GPU needed): the library loads, exports every symbol that
include/btd.h declares, and the plan's symbolic analysis (a0) agrees with the oracle's plain
definitions of P_inf, level counts and the coupling-slot layout."""
import os
import re

import pytest
import torch

import paper_2601_03754_b200 as btd
from oracle.perm import coupling_slots, num_levels, perm

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "btd.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(btd_[a-z_0-9]+)\s*\(", src)))


@pytest.fixture(scope="module", autouse=True)
def _built():
    from paper_2601_03754_b200 import build

    build.build()


def test_exports_every_declared_symbol():
    names = _declared_symbols()
    assert len(names) >= 15
    L = btd.lib()
    for name in names:
        assert hasattr(L, name), name
    # the binding wires every declared entry point
    assert {s[0] for s in btd.btd.SIGNATURES} == set(names)


def test_shared_object_is_sm100a():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", btd.btd.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("N", [1, 2, 3, 4, 5, 7, 8, 9, 16, 17, 20, 33, 64, 100, 128, 256, 1000, 1024, 4096])
def test_plan_matches_oracle_definitions(N):
    p = btd.Plan(N, 3, 2, 1, torch.float64)
    assert p.levels == num_levels(N)
    slots = coupling_slots(N)
    assert p.num_coupling_blocks == len(slots)
    for lev in range(1, p.levels + 2):
        assert p.level_offset(lev) == sum(1 for s in slots if s[0] < lev)
    assert p.level_offset(0) == -1 and p.level_offset(p.levels + 2) == -1
    assert p.permutation() == [i - 1 for i in perm(N)]


def test_variant_selection():
    # c5 (n=12, N=128, fp32) fits one SM's shared memory -> fused; single long systems with
    # n <= 32 whose column ops fit 4 CTAs per SM -> wide (c2, c3); n > 32 -> persist (c4)
    assert btd.Plan(128, 12, 8192, 1, torch.float32).variant == "fused"
    assert btd.Plan(1024, 32, 1, 1, torch.float64).variant == "wide"
    assert btd.Plan(4096, 32, 1, 1, torch.float64).variant == "wide"     # <= 2048 level-1 columns (fp64)
    assert btd.Plan(8192, 32, 1, 1, torch.float64).variant == "persist"
    assert btd.Plan(2048, 32, 1, 1, torch.float32).variant == "wide"     # <= 1024 (fp32)
    assert btd.Plan(4096, 32, 1, 1, torch.float32).variant == "persist"
    assert btd.Plan(8192, 32, 1, 65, torch.float64).variant == "wide"    # many right-hand sides
    assert btd.Plan(1000, 32, 4, 1, torch.float64).variant == "wide"     # batched fp64 n=32: <= 2048 columns
    assert btd.Plan(1024, 16, 4, 1, torch.float64).variant == "persist"  # other batched: 4 x 148 columns
    assert btd.Plan(1000, 32, 3, 1, torch.float32).variant == "persist"
    assert btd.Plan(256, 128, 1, 1, torch.float64).variant == "persist"
    assert btd.Plan(64, 16, 1, 1, torch.float64).variant == "wide"
    assert btd.Plan(8, 16, 1, 1, torch.float64).variant == "fused"
    assert btd.Plan(8, 32, 1, 1, torch.float64).variant == "wide"       # 32-wide blocks: from N = 4 (fp64)
    assert btd.Plan(8, 32, 1, 1, torch.float32).variant == "fused"      # ... and N = 12 (fp32)
    assert btd.Plan(12, 32, 1, 1, torch.float32).variant == "wide"
    # one short system with small blocks: the one-CTA FUSED kernel (no grid barriers) wins
    assert btd.Plan(512, 4, 1, 1, torch.float64).variant == "fused"
    assert btd.Plan(64, 12, 1, 1, torch.float64).variant == "fused"
    assert btd.Plan(128, 12, 1, 1, torch.float64).variant == "wide"
    assert btd.Plan(128, 12, 1, 1, torch.float32).variant == "fused"
    assert btd.Plan(128, 12, 8, 1, torch.float32).variant == "fused"      # <= 148 systems: all CTAs at once
    assert btd.Plan(128, 16, 4, 1, torch.float64).variant == "wide"
    assert btd.Plan(8, 2, 1, 1, torch.float64).launches() == 1
    assert btd.Plan(1024, 32, 1, 1, torch.float64).launches() == 1
    p = btd.Plan(1024, 32, 1, 1, torch.float64, variant="level")
    assert p.launches("factor_solve") == 1 + 2 * p.levels
    with pytest.raises(btd.BtdError):
        btd.Plan(256, 64, 1, 1, torch.float64, variant="level")
    with pytest.raises(btd.BtdError):
        btd.Plan(8192, 32, 1, 1, torch.float64, variant="fused")


@pytest.mark.parametrize("args", [(0, 4, 1, 1), (4, 0, 1, 1), (4, 4, 0, 1), (4, 4, 1, 0)])
def test_plan_rejects_bad_sizes(args):
    with pytest.raises(btd.BtdError):
        btd.Plan(*args, dtype=torch.float32)


def test_unsupported_block_size():
    with pytest.raises(btd.BtdError):
        btd.Plan(8, 200, 1, 1, torch.float64)


def test_cpu_tensors_are_rejected():
    """No CPU fallback: host tensors are refused before any launch."""
    D = torch.eye(2, dtype=torch.float64).expand(1, 4, 2, 2).contiguous()
    E = torch.zeros(1, 3, 2, 2, dtype=torch.float64)
    with pytest.raises(btd.BtdError):
        btd.factor(D, E)


def test_status_strings():
    L = btd.lib()
    assert L.btd_status_string(0) == b"BTD_OK"
    assert b"invalid" in L.btd_status_string(1)


def test_auto_rejects_oversized_persist_at_plan_time():
    """n = 128 fp64 with 256 right-hand sides needs more than 227 KB of shared memory in PERSIST:
    AUTO refuses at plan creation (BTD_EUNSUPPORTED) instead of failing at every launch."""
    import ctypes

    L = btd.lib()
    h = ctypes.c_void_p()
    assert L.btd_plan_create(ctypes.byref(h), 256, 128, 1, 256, 1) == 4
    assert L.btd_plan_create(ctypes.byref(h), 256, 128, 1, 1, 1) == 0
    L.btd_plan_destroy(h)


def test_misaligned_device_pointers_are_rejected_before_launch():
    """Every device buffer is accessed with 16-byte vector operations from its base: a misaligned
    pointer returns BTD_EINVAL (checked on the host, before any CUDA call -- no GPU needed)."""
    import ctypes

    L = btd.lib()
    p = btd.Plan(8, 4, 1, 1, torch.float32)
    a, mis = ctypes.c_void_p(1 << 20), ctypes.c_void_p((1 << 20) + 4)
    st = ctypes.c_void_p(0)
    assert L.btd_factor(p.handle, mis, a, a, a, a, st) == 1
    assert L.btd_factor(p.handle, a, a, a, mis, a, st) == 1
    assert L.btd_factor(p.handle, a, a, a, a, ctypes.c_void_p((1 << 20) + 2), st) == 1
    assert L.btd_solve(p.handle, a, a, mis, a, st) == 1
    assert L.btd_factor_solve(p.handle, a, a, a, a, a, mis, a, st) == 1
    args = [a] * 7 + [a, a, a, a, a, mis, a]
    assert L.btd_factor_solve_host(p.handle, *args, 1, st) == 1


def test_binding_checks_caller_supplied_outputs():
    """out= buffers go through the same shape/dtype/device checks as the inputs (before any launch)."""
    D = torch.eye(2, dtype=torch.float64).expand(1, 4, 2, 2).contiguous()
    E = torch.zeros(1, 3, 2, 2, dtype=torch.float64)
    b = torch.ones(1, 4, 2, 1, dtype=torch.float64)
    with pytest.raises((btd.BtdError, ValueError, TypeError)):
        btd.factor_solve(D, E, b, out=(D, E, b, torch.zeros(1, dtype=torch.int32)))
    ws_plan = btd.Plan(4, 2, 1, 1, torch.float64)
    with pytest.raises(ValueError):
        btd.btd._check_host("D", torch.zeros(1, 4, 2, 3, dtype=torch.float64), (1, 4, 2, 2), torch.float64)
    assert ws_plan.num_coupling_blocks == 4


def _v2(o):
    return (o & -o).bit_length() - 1


def _r2_cache_plan(N):
    """Host mirror of R2Cache (csrc/btd_fused_r2.cuh): first cached level LC and the odd slot of
    every cached coupling block, handed out in order of death."""
    L = N.bit_length()
    NO = (N + 1) // 2
    ccount = lambda l: (N >> (l - 1)) - 1
    group = lambda g: ((NO - 1) >> g) // 2 + ((NO - 1) >> g) % 2
    LC = L + 1
    for lc in range(3, L + 1):
        need, ok = 0, True
        for l in range(lc, L + 1):
            need += ccount(l)
            if need > sum(group(g) for g in range(0, l - 2)):
                ok = False
                break
        if ok:
            LC = lc
            break
    order = []
    g = 0
    while len(order) < NO:
        cnt = group(g)
        order += [(2 * q + 1) << g for q in range(cnt)]
        g += 1
        if g > 40:
            break
    return LC, order


@pytest.mark.parametrize("N", list(range(1, 70)) + [100, 127, 128, 129, 255, 256, 1000, 1024, 4096])
def test_fused_r2_slot_schedule_is_race_free(N):
    """FUSED-R2's shared-memory schedule, simulated level by level on the host: every fill lands in
    a free odd slot and is read exactly once by the next level's column (Alg. 4 l.13 -> l.10/l.12);
    backward-cache entries of level l >= LC land in odd slots that are dead for the rest of the
    factorization (never holding a fill that is still to be read, never overwritten later)."""
    L = N.bit_length()
    LC, order = _r2_cache_plan(N)
    live = {}  # odd slot index -> ("fill", level) or ("cache", level)
    q = 0
    for l in range(1, L + 1):
        s = 1 << (l - 1)
        cols = list(range(s, N + 1, 2 * s))
        if l >= LC:  # cache entries of this level: coupling blocks k = 1..N/s-1
            for _ in range(ccount := (N >> (l - 1)) - 1):
                o = order[q]
                assert o not in live, (N, l, o, live.get(o))
                live[o] = ("cache", l)
                q += 1
        for c in cols:
            hasL, hasR = c > s, c + s <= N
            if l >= 2:
                if hasL:
                    assert live.pop((c - s) // 2) == ("fill", l - 1)
                if hasR:
                    assert live.pop(c // 2) == ("fill", l - 1)
            if hasL and hasR:
                o = (c - s) // 2  # odd slot of block c - s + 1
                assert o not in live
                live[o] = ("fill", l)
    assert all(v[0] == "cache" for v in live.values())
    if N == 128:
        assert LC == 3


def test_extension_entry_points_validate_before_launch():
    """§8(f) entry points (csrc/btd_ext.cu) reject bad arguments on the host, without a GPU."""
    import ctypes

    L = btd.lib()
    p64 = btd.Plan(16, 4, 2, 1, torch.float64)
    p32 = btd.Plan(16, 4, 2, 1, torch.float32)
    sz = ctypes.c_size_t(0)
    assert L.btd_mixed_workspace_bytes(p64.handle, ctypes.byref(sz)) == 1          # needs a binary32 plan
    assert L.btd_mixed_workspace_bytes(p32.handle, ctypes.byref(sz)) == 0
    nn, nx = 16, 2 * 16 * 4
    expect = sum(((v + 255) // 256) * 256 for v in (2 * 16 * nn * 4, 2 * 15 * nn * 4, nx * 4, nx * 4, nx * 8, 2 * 2 * 8))
    assert sz.value == expect
    fake = ctypes.c_void_p(4096)  # never dereferenced: every call below fails its checks first
    # mixed: iters < 0, misaligned x
    assert L.btd_mixed_factor_solve(p32.handle, fake, fake, fake, fake, fake, fake, fake, -1, None, fake, None) == 1
    assert L.btd_mixed_factor_solve(p32.handle, fake, fake, fake, fake, fake, ctypes.c_void_p(4100), fake, 1, None,
                                    fake, None) == 1
    # arrow: na must leave at least one rhs column (plan m = na + mb)
    pa = btd.Plan(16, 4, 2, 3, torch.float64)
    assert L.btd_arrow_factor_solve(pa.handle, 3, *([fake] * 14), None) == 1
    assert L.btd_arrow_factor_solve(pa.handle, 0, *([fake] * 14), None) == 1
    # banded: the plan must be the super-block plan (ceil(N/w), w n)
    pb = btd.Plan(5, 12, 1, 1, torch.float64)
    assert L.btd_banded_factor_solve(pb.handle, 13, 4, 2, *([fake] * 11), None) == 1
    assert L.btd_banded_factor_solve(pb.handle, 16, 4, 3, *([fake] * 11), None) == 1
    # partition: batch must be 1; reduce needs p >= 2 and a plan of p - 1 blocks
    assert L.btd_partition_local(p64.handle, *([fake] * 13), None) == 1
    ps = btd.Plan(3, 4, 1, 1, torch.float64)
    assert L.btd_partition_reduce(ps.handle, 3, *([fake] * 8), None) == 1
    assert L.btd_partition_reduce(ps.handle, 1, *([fake] * 8), None) == 1
    pc = btd.Plan(8, 4, 1, 1, torch.float64)
    assert L.btd_partition_finish(pc.handle, fake, fake, None, fake, None) == 1    # m = 1 - n < 1
