"""The shape -> kernel-configuration table (gemm_api.cu pick_config; the paper's per-size
"best performing version"), evaluated on the host for the B200's 148 SMs.

Every expectation below is a measured winner (profiles/r01: cfgsweep.md, wide_tile.md,
f32_short_k_cfg.txt, multicast.md, splitk.md v8/v9, mid_size_configs.txt; profiles/r02:
graph_small_pick*.jsonl for the split-K thresholds).  The F32 chain
limit of the split-K configs (R4/R17) is checked as an invariant over a grid."""
import itertools

import pytest

import paper_2108_13191_b200 as g

SM = 148
C = g.CONFIGS

CASES = [
    # (M, N, K, acc, expected config name)
    (8192, 8192, 8192, 0, "pair_256x256_k128"),      # bench F32
    (8192, 8192, 8192, 1, "pair_256x512"),           # bench F16: the wide tile
    (16384, 16384, 16384, 1, "pair_256x512"),
    (4096, 4096, 4096, 1, "pair_256x512"),
    (2048, 2048, 2048, 1, "pair_256x256_s4"),        # one wave: 3 staging slots pipeline the stores
    (2048, 2048, 2048, 0, "pair_256x256_s4"),
    (1536, 3072, 2048, 0, "pair_256x256_s4"),
    (2048, 2048, 4096, 1, "pair_256x256_s4"),
    (2048, 2048, 8192, 0, "pair_256x256_k128"),      # ... but not at K = 8192
    (2560, 2048, 2048, 0, "pair_256x256"),           # 80 pair tiles: more than one wave
    (2304, 2304, 2304, 0, "pair_256x256_s4"),        # r02: F32 just over one wave, stream-K: S4
    (2304, 2560, 2560, 0, "pair_256x256_s4"),
    (2304, 2304, 4096, 0, "pair_256x256_s4"),
    (2304, 2304, 8192, 0, "pair_256x256_k128"),      # ... not at K = 8192
    (2560, 2560, 2560, 0, "pair_256x256_k128"),      # ... nor at 100 tiles (1.35 waves)
    (3072, 3072, 2048, 1, "pair_256x512"),
    (2304, 2304, 2304, 1, "pair_256x256_k128"),      # F16: stream-K over the partial last wave
    (2560, 2560, 8192, 1, "pair_256x256_k128"),
    (4608, 4608, 4608, 1, "pair_256x256_k128"),
    (4096, 4096, 4096, 0, "pair_256x256_k128"),      # F32 (stream-K is decided at launch)
    (1792, 1792, 8192, 1, "pair_256x256_k128"),      # F16 below one wave, long K: stream-K
    (1792, 1792, 4096, 1, "pair_256x256_s4"),        # (one wave, K <= 4096: the 3-slot config)
    (32768, 1024, 4096, 1, "pair_256x256_k128"),
    (16384, 4096, 1024, 0, "pair_256x256"),          # F32 one K chunk, reduce-add epilogue
    (8192, 1002, 1000, 0, "pair_256x256_s5"),        # ... but a ragged N (N % 4 != 0) still stages C_in
    (1024, 1024, 1024, 0, "solo_128x64"),            # r02: the two-way split loses below K = 4096
    (1024, 1024, 1024, 1, "solo_128x64"),
    (2048, 1024, 1024, 0, "solo_128x128"),           # at most half a wave of pair tiles
    (256, 1024, 16384, 1, "splitk_128x128_s4"),      # small output, long K
    (512, 512, 8192, 0, "splitk_128x128_s4"),
    (1024, 1024, 4096, 0, "splitk_128x128_s2"),      # r02: F32 S2 x 128x128 at K = 4096 ...
    (1024, 1024, 8192, 0, "splitk_128x256_s4"),      # ... S4 x 128x256 from K = 8192
    (1024, 1024, 4096, 1, "splitk_128x128_s2"),      # F16: the bulk-DMA S2 configs
    (1024, 1024, 8192, 1, "splitk_128x128_s2"),
    (1024, 1024, 16384, 1, "splitk_128x256_s4"),
    (1024, 2048, 4096, 0, "solo_128x128"),           # r02: 17.7 vs 19.2 us for S2 x 128x256
    (2048, 1024, 4096, 1, "solo_128x128"),           # r02: 17.9 vs 21.7 us
    (1024, 1024, 2048, 0, "solo_128x64"),            # r02: 9.1 vs 10.0 us split
    (1024, 1024, 2048, 1, "solo_128x64"),            # r02: 8.8 vs 10.8 us split
    (1024, 512, 1024, 0, "solo_128x64"),
    (768, 768, 2048, 0, "solo_128x64"),
    (768, 768, 2048, 1, "solo_128x64"),
    (768, 768, 4096, 0, "splitk_128x128_s2"),        # 36 x 4 CTAs would not fit in 4-CTA clusters
    (768, 768, 4096, 1, "splitk_128x128_s2"),
    (2048, 1024, 2048, 0, "solo_128x128"),           # r02: 11.7 vs 13.8 us for S2 x 128x256
    (512, 512, 1024, 1, "solo_128x64"),              # S2 only from K = 4096
]


@pytest.mark.parametrize("M,N,K,acc,want", CASES)
def test_measured_winners(M, N, K, acc, want):
    assert g.pick_config(M, N, K, acc, sm_count=SM) == C[want], (M, N, K, acc)


def test_f32_split_chain_never_exceeds_4096():
    # each split CTA keeps one truncating TMEM chain over K / S: for F32 C it must stay
    # <= 4096 long (rel. error ~5e-6 against the 1e-5 bar); F16 has no such limit
    splits = {C["splitk_128x256_s2"]: 2, C["splitk_128x256_s4"]: 4, C["splitk_128x128_s4"]: 4,
              C["splitk_128x128_s2"]: 2}
    seen = set()
    for M, N, K in itertools.product([64, 128, 256, 512, 1024, 2048], [64, 256, 512, 1024, 2048, 4096],
                                     [1024, 2048, 4096, 8192, 16384, 32768, 65536]):
        for acc in (0, 1):
            cfg = g.pick_config(M, N, K, acc, sm_count=SM)
            assert cfg > 0
            if cfg in splits:
                seen.add((acc, cfg))
                if acc == 0:
                    assert -(-K // splits[cfg]) <= 4096, (M, N, K, cfg)
    assert {(0, C["splitk_128x128_s4"]), (1, C["splitk_128x128_s4"])} <= seen


def test_bad_arguments():
    assert g.pick_config(8, 8, 8, 7, sm_count=SM) == -1
    assert g.pick_config(8, 8, 8, 0, sm_count=1) == -1
