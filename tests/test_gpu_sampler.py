"""GPU: the sm_100a Philox + Floyd sampler is bit-exact with the reference
generate_masks (sampler.cpp:153-210) — golden fixtures, the compiled reference,
and size-independent properties at BASELINE sizes."""
import numpy as np
import pytest

import paper_2506_22668_b200 as sf
from conftest import hex_to_u64

pytestmark = pytest.mark.gpu


def test_device_philox_golden(ctx, golden):
    for c in golden["philox"]:
        got = ctx.philox(c["seed"], c["stream"], len(c["out"]))
        assert (got == hex_to_u64(c["out"])).all()
    # SURVEY.md Appendix A
    assert [f"{x:016x}" for x in ctx.philox(0x0123456789ABCDEF, 7, 3)] == [
        "a6c02cf2fdbf9305", "8ec43d2634b23a77", "c59490403ec6e16d"]


def test_masks_golden(ctx, golden):
    for c in golden["masks"]:
        p = sf.plan_sizes(c["n"], c["k"], c["allow"])
        bits, ros = ctx.generate_masks(p, int(c["seed"], 16), c["rank"], c["world"])
        assert list(bits.shape) == c["shape"]
        assert (bits.ravel() == hex_to_u64(c["bits"])).all()
        assert ros.tolist() == c["rows_of_size"]


def test_appendix_a_rows(ctx):
    p = sf.plan_sizes(12, 1000, False)
    bits, _ = ctx.generate_masks(p, 42)
    assert [hex(int(x)) for x in bits[:6, 0]] == ["0x2", "0xffd", "0x10", "0xfef", "0x400", "0xbff"]
    bits3, _ = ctx.generate_masks(p, 42, 3, 8)
    assert bits3.shape[0] == 126 and int(bits3[0, 0]) == 0x20


@pytest.mark.parametrize("n,k,allow,seed,world", [
    (999, 10000, True, 0x516F7AECD40A0D17, 1),    # C1 shape, full
    (70, 2000, False, 11, 1),                      # two words, tail bits
    (64, 4000, False, 3, 1),                       # exact word boundary
    (4, 20, True, 7, 1),                           # exhaustive (test_sampler.cpp:119-142)
    (9, 1022, True, 3, 4),                         # exhaustive, sharded
    (30, 25000, True, 9, 4),                       # acceptance c5
    (3000, 4000, False, 77, 3),                    # sharded, mid n
])
def test_masks_bit_exact_vs_reference(ctx, ref, n, k, allow, seed, world):
    p = sf.plan_sizes(n, k, allow)
    for rank in range(world):
        got, ros = ctx.generate_masks(p, seed, rank, world)
        want, wros = ref.generate_masks(n, k, seed, rank, world, allow_exhaustive=allow)
        assert got.shape == want.shape
        assert (got == want).all()
        assert (ros == wros).all()


def test_large_n_global_memory_path_vs_port(ctx, port):
    # n = 400,000 players exceeds the shared-memory bitset budget and takes
    # the global-memory Floyd path; check a slice of pairs bit-for-bit
    n, k = 400_000, 256
    p = sf.plan_sizes(n, k, False)
    got, _ = ctx.generate_masks(p, 5)
    pp = port.plan_sizes(n, k, False)
    want = port.generate_masks(n, pp, 5, 0, 1, 0, 24)
    assert (got[:48] == want).all()


def test_c2_shard_properties_and_slices(ctx, port):
    """BASELINE config C2 (n = 49,648, k = 500K): full rank-0-of-8 shard on the
    GPU; bit-exact against the port on slices spread over the size classes, and
    size-independent properties on every row (complements, class sizes)."""
    n, k, world, seed = 49_648, 500_000, 8, 0x1234
    p = sf.plan_sizes(n, k, True)
    bits, ros = ctx.generate_masks(p, seed, 0, world)
    pairs = bits.shape[0] // 2
    W = (n + 63) // 64
    tail = (1 << (n % 64)) - 1
    even, odd = bits[0::2], bits[1::2]
    assert ((odd[:, :-1] == ~even[:, :-1])).all()
    assert (odd[:, -1] == (~even[:, -1] & np.uint64(tail))).all()
    pc = np.unpackbits(even.view(np.uint8), axis=1).sum(1)
    g = np.arange(pairs, dtype=np.uint64) * world
    cls = np.searchsorted(p["first"], g, side="right") - 1
    assert (pc == p["sizes"][cls]).all()
    pp = port.plan_sizes(n, k, True)
    total = int(pp["first"][-1] + pp["pairs"][-1])
    for g0 in [0, 200_000, 248_000, 249_900]:
        want = port.generate_masks(n, pp, seed, 0, world, g0, min(total, g0 + 8 * 24))
        j0 = (g0 + world - 1) // world  # first local pair (rank 0) at or after g0
        assert (bits[2 * j0: 2 * j0 + want.shape[0]] == want).all()
    assert bits.shape[1] == W
