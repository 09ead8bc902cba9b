"""Register budget of the shipped kernels (CPU; reads the ptxas -v log the build writes to
paper_2108_13191_b200/csrc/ptxas_info.txt): the data-parallel pair and 1-CTA kernels and the
256 x 512 F16 kernel must not spill -- their epilogues run at the 168-register limit of
352 threads per SM, and a spill there lands in the drain the MMA waits on (round 2 measured a
shuffle-based bias staging that pushed 24 instantiations into spills, and reverted it)."""
import os
import re

import pytest

LOG = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2108_13191_b200", "csrc",
                   "ptxas_info.txt")

# mangled-name fragments of the kernels AUTO picks for the plain C += A.B (SK = false builds)
SHIPPED = {
    "pair_256x256_k128 F32": "KCfgILi2ELi256ELi3ELb0ELi1ELi128ELb0ELi1ELb1EEELb0EE",
    "pair_256x256_k128 F16": "KCfgILi2ELi256ELi3ELb1ELi1ELi128ELb0ELi1ELb1EEELb0EE",
    "pair_256x256 F32": "KCfgILi2ELi256ELi6ELb0ELi1ELi64ELb0ELi1ELb1EEELb0EE",
    "pair_256x256_s4 F32": "KCfgILi2ELi256ELi4ELb0ELi3ELi64ELb0ELi1ELb1EEELb0EE",
    "pair_256x256_s5 F32": "KCfgILi2ELi256ELi5ELb0ELi2ELi64ELb0ELi1ELb1EEELb0EE",
    "solo_128x64 F16": "KCfgILi1ELi64ELi8ELb1ELi1ELi64ELb0ELi1ELb1EEELb0EE",
    "solo_128x128 F32": "KCfgILi1ELi128ELi6ELb0ELi1ELi64ELb0ELi1ELb1EEELb0EE",
    "pair_256x512 F16": "gemm_f16_sm100_wide_kernelINS_4WCfgILi4EEELb0EE",
}


def _spills():
    with open(LOG) as f:
        txt = f.read()
    out = {}
    for block in re.split(r"ptxas info    : Compiling entry function '", txt)[1:]:
        name = block.split("'")[0]
        m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", block)
        out[name] = (int(m.group(1)), int(m.group(2))) if m else (0, 0)
    return out


@pytest.mark.skipif(not os.path.exists(LOG), reason="no ptxas log (run __graft_entry__.build())")
@pytest.mark.parametrize("what", sorted(SHIPPED))
def test_shipped_kernels_do_not_spill(what):
    sp = _spills()
    hits = [v for k, v in sp.items() if SHIPPED[what] in k]
    assert hits, f"{what}: kernel not found in the ptxas log"
    assert all(v == (0, 0) for v in hits), f"{what}: spills {hits}"
