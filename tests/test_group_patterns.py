"""The row-group kernel's static pattern library (csrc/group_patterns.hpp) against the
oracle's topological-insulator generator (models.cpp:80-139): for sites away from the x / y
wrap, the merged column list of a site's four rows must have exactly the library's row
masks, own-row position and purely-real / purely-imaginary entry classes (bottom plane,
interior and top plane of the slab).  A library that drifted from the generator would only
cost speed (the device builder compares per group and falls back to the generic path), but
this pins it on the CPU."""
import os
import re

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "paper_1510_04895_b200", "csrc", "group_patterns.hpp")


def library():
    text = open(HDR).read()
    out = {}
    for name in ("PatTiMid", "PatTiLo", "PatTiHi"):
        body = text[text.index(f"struct {name} "):]
        body = body[:body.index("\n};")]
        nc, own = map(int, re.search(r"NC = (\d+), OWN = (\d+)", body).groups())
        tabs = {}
        for fn in ("m", "re", "im"):
            m = re.search(rf"constexpr unsigned {fn}\(int k\) \{{\s*constexpr unsigned char t\[NC\] = \{{([^}}]*)\}}",
                          body)
            tabs[fn] = [int(x, 16) for x in m.group(1).replace("\n", " ").split(",")]
            assert len(tabs[fn]) == nc
        out[name] = (nc, own, tabs)
    return out


def site_pattern(csr, g):
    offs, cols, vals = csr.offs, csr.cols, csr.vals
    rows = [dict(zip(cols[offs[r]:offs[r + 1]].tolist(), vals[offs[r]:offs[r + 1]].tolist()))
            for r in range(4 * g, 4 * g + 4)]
    union = sorted(set().union(*rows))
    mask = [sum(1 << r for r in range(4) if c in rows[r]) for c in union]
    re_ = [sum(1 << r for r in range(4) if c in rows[r] and rows[r][c].imag == 0) for c in union]
    im_ = [sum(1 << r for r in range(4) if c in rows[r] and rows[r][c].real == 0) for c in union]
    return union, mask, re_, im_


def test_library_patterns_match_the_oracle_generator(orc):
    lx, ly, lz = 6, 5, 4
    csr = orc.topological_insulator(lx, ly, lz, disorder=0.5, seed=1)
    lib = library()
    seen = {k: 0 for k in lib}
    for z in range(lz):
        name = "PatTiLo" if z == 0 else ("PatTiHi" if z == lz - 1 else "PatTiMid")
        nc, own, tabs = lib[name]
        for y in range(1, ly - 1):
            for x in range(1, lx - 1):
                g = x + lx * (y + ly * z)
                union, mask, re_, im_ = site_pattern(csr, g)
                assert len(union) == nc
                assert mask == tabs["m"]
                assert union[own:own + 4] == [4 * g + r for r in range(4)]
                # every entry the library multiplies as purely real / imaginary is so
                for k in range(nc):
                    assert tabs["re"][k] & ~re_[k] == 0 and tabs["im"][k] & ~im_[k] == 0
                    assert tabs["re"][k] & tabs["im"][k] == 0
                    assert (tabs["re"][k] | tabs["im"][k]) & ~mask[k] == 0
                seen[name] += 1
    assert all(v > 0 for v in seen.values())
    # the library classifies every entry of these sites (none is left to the 4-multiply form)
    for name, (nc, own, tabs) in lib.items():
        assert [a | b for a, b in zip(tabs["re"], tabs["im"])] == tabs["m"]


def pair_rule():
    """pair_col / pair_neg of PatBase (group_patterns.hpp) restated: positions after the z-1
    columns, and the sign table's bit mask."""
    text = open(HDR).read()
    mask = int(re.search(r"return \((0x[0-9A-Fa-f]+)u >> \(k - \(D::OWN - 8\)\)\) & 1u;", text).group(1), 16)
    assert "(q >= 0 && q < 8) || (q >= 12 && q < 20)" in text

    def pair_col(k, own, m):
        q = k - (own - 8)
        return ((0 <= q < 8) or (12 <= q < 20)) and m in (0x3, 0xC)

    def pair_neg(k, own):
        return (mask >> (k - (own - 8))) & 1
    return pair_col, pair_neg


def test_row_pair_products_match_the_oracle_generator(orc):
    """The site-ring kernel multiplies an x / y neighbour column ONCE for the two rows of a
    row pair (step_ring.cuh ring_mac): the two values must be +-v / +-iv of one magnitude
    with the relative sign of PatBase::pair_neg (hop[j] = -t (G1 - i G^{j+1}) / 2,
    models.cpp:88-93), for every static site, whatever t and the disorder are; every x / y
    neighbour column must be such a pair column, the z and own columns never."""
    pair_col, pair_neg = pair_rule()
    lib = library()
    lx, ly, lz = 6, 5, 4
    for kw in (dict(disorder=0.5, seed=1), dict(disorder=0.0, seed=3)):
        csr = orc.topological_insulator(lx, ly, lz, **kw)
        offs, cols, vals = csr.offs, csr.cols, csr.vals
        checked = 0
        for z in range(lz):
            name = "PatTiLo" if z == 0 else ("PatTiHi" if z == lz - 1 else "PatTiMid")
            nc, own, tabs = lib[name]
            for y in range(1, ly - 1):
                for x in range(1, lx - 1):
                    g = x + lx * (y + ly * z)
                    rows = [dict(zip(cols[offs[r]:offs[r + 1]].tolist(), vals[offs[r]:offs[r + 1]].tolist()))
                            for r in range(4 * g, 4 * g + 4)]
                    union = sorted(set().union(*rows))
                    for k, c in enumerate(union):
                        site = c // 4 - g
                        is_xy = site in (-1, 1, -lx, lx)
                        assert pair_col(k, own, tabs["m"][k]) == is_xy, (name, k)
                        if not is_xy:
                            continue
                        ra = 0 if tabs["m"][k] == 0x3 else 2
                        va, vb = rows[ra][c], rows[ra + 1][c]
                        # the component each product uses: real part of a purely real value,
                        # imaginary part of a purely imaginary one
                        ca = va.imag if (tabs["im"][k] >> ra) & 1 else va.real
                        cb = vb.imag if (tabs["im"][k] >> (ra + 1)) & 1 else vb.real
                        assert ca != 0.0 and cb == (-ca if pair_neg(k, own) else ca), (name, k, va, vb)
                        checked += 1
        assert checked == 16 * (lx - 2) * (ly - 2) * lz
