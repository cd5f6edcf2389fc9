"""GPU: block- and device-level collaborative conversion of long numeric fields.

Numeric fields of >= 1 KB without inner control bytes are converted by one thread block each; fields of
>= 256 KB by the whole grid.  Every value / valid byte must equal the oracle's (strtod / exact int64),
through every entry point (plan, parse_into, library-owned; k_small below 2 MB, the staged kernels above),
and the stats must show which tier ran."""
import random

import numpy as np
import pytest

import oracle
from tests.gpu_helpers import compare

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
import paper_1905_13415_b200 as parpa  # noqa: E402

TYPES = [oracle.INT64, oracle.FLOAT64, oracle.SPAN]


def dev(data):
    a = np.frombuffer(bytes(data), np.uint8)
    t = torch.empty(max(a.size, 1), dtype=torch.uint8, device="cuda")
    if a.size:
        t[:a.size].copy_(torch.from_numpy(a.copy()))
    return t[:a.size]


def long_ints(rng, L):
    z = "0" * L
    return [z + "123", "-" + z + "9223372036854775808", z + "9223372036854775807", z + "9223372036854775808",
            "1" * L, z + "x", "+" + z, "-" + z, z[:L // 2] + "-" + z[L // 2:], z + "12.5", "+-" + z + "1",
            "".join(rng.choice("0123456789") for _ in range(L)), z + "1e5", z[:-1] + "+"]


def long_floats(rng, L):
    z = "0" * L
    d = "".join(rng.choice("0123456789") for _ in range(L))
    return ["0." + z + "123e" + str(L + 5), "1" * L, "1" * L + "." + "9" * L, z + "." + z, "-" + z, "-" + z + "." + z,
            "1" * 800 + "5" + "0" * L, "1" * 799 + "5" + "0" * L + "1", "4" * 800 + "5" + z,
            "2" * L + "e-" + z + "1500", d + "." + d + "E+" + z + "7", "." + d, d + ".", "-." + d + "e-" + str(L // 3),
            # invalid grammar
            "1.2." + z, z + "e5e6", z + "1e", "." + z[:-1] + "." , "e" + "1" * L, "1" * L + "e+-5", z + " ",
            "+" + d + "e" + "-" * 2 + "3", "." * L,
            # exponents far beyond the significand (saturation must not flip the result)
            "1" + z + "e-" + "9" * 15, "1" + z + "e+" + "9" * 15, z + "e" + "9" * 40]


def build_rows(rng, L, nfill=200):
    """Ordinary short records around records whose int / float field is long."""
    rows = []
    for i in range(nfill):
        rows.append(f"{i},{i * 0.25},s{i}")
    for s in long_ints(rng, L):
        rows.append(f"{s},1.5,i{L}")
        rows.append(f"{rng.randint(-99, 99)},2.5,x")
    for s in long_floats(rng, L):
        rows.append(f"7,{s},f{L}")
        rows.append(f"{rng.randint(-99, 99)},0.125,y")
    for i in range(nfill):
        rows.append(f"{-i},{i}.5e-3,t{i}")
    return ("\n".join(rows) + "\n").encode()


def run_paths(data, label):
    schema = parpa.Schema(list(TYPES))
    ora = oracle.parse("csv", data, len(TYPES), list(TYPES))
    d = dev(data)
    dfa = parpa.Dfa.dialect("csv")
    res = parpa.parse(dfa, schema, d)
    compare(res, ora, TYPES, label + "/plan")
    cap = max(ora.R, 1) + 3
    cols = parpa.alloc_columns(schema, cap)
    st = parpa.new_stats_tensor()
    parpa.parse_into(dfa, schema, d, cols, cap, st)
    stats = parpa.stats_from_tensor(st)
    compare(parpa.ParseResult(cols, stats), ora, TYPES, label + "/into")
    compare(parpa.parse_c_owned(dfa, schema, d), ora, TYPES, label + "/owned")
    return stats


@pytest.mark.parametrize("L", [1024, 1500, 5000, 70_000])
def test_block_tier_long_numbers(L):
    rng = random.Random(L)
    data = build_rows(rng, L)
    stats = run_paths(data, f"block-{L}")
    assert stats["block_fields"] > 0, stats
    if len(data) > 2_000_000:                      # staged kernels (k_small below 2 MB)
        assert stats["device_fields"] == 0, stats


@pytest.mark.parametrize("L", [300_000, 1_200_000])
def test_device_tier_huge_numbers(L):
    rng = random.Random(L)
    z = "0" * L
    rows = ["1,2,a"] * 500
    for s in [z + "42", "9" * L, "-" + z + "9223372036854775807", z + "x1"]:
        rows += [f"{s},0.5,i", "3,4,b"]
    for s in ["1" + z[:-10] + "e-" + str(L - 10), "0." + z + "25", z + "." + "3" * L, "1" * L,
              "-" + z, "1" + z + "e-" + "9" * 15, z + "..5", "5" * 900 + "0" * L + "1"]:
        rows += [f"5,{s},f", "6,7.75,c"]
    rows += ["8,9,z"] * 500
    data = ("\n".join(rows) + "\n").encode()
    stats = run_paths(data, f"device-{L}")
    assert stats["device_fields"] > 0 and stats["block_fields"] >= 0, stats


def test_collab_fields_in_small_and_staged_paths():
    """the same long fields inside an input below 2 MB (the cooperative k_small kernel) and above it"""
    rng = random.Random(7)
    small = build_rows(rng, 3000, nfill=100)
    assert len(small) < 2_000_000
    st = run_paths(small, "small")
    assert st["block_fields"] > 0, st
    pad = ("\n".join(f"{i},{i}.25,p" for i in range(200_000)) + "\n").encode()
    big = pad + small + pad
    assert len(big) > 2_000_000
    st = run_paths(big, "staged")
    assert st["block_fields"] > 0, st
