"""Block-granular LRU model of the operand DRAM traffic of the persistent pair-tile schedule
(8192^3, 256 x 256 pair tiles, 74 clusters, tile_coords' grouped raster): every wave's tiles
step through K in lockstep, each k-block reads one 32 KB A block and one 32 KB B block; a miss
in an LRU of `cap_mb` is a DRAM read.  Used to read the measured DRAM traffic
(profiles/r02/findings.md section 9); not a product component.
usage: python tools/l2_reuse_model.py"""
import collections, sys
def tile_coords(tile, tiles_m, tiles_n, group_m, snake=False):
    per_group = group_m * tiles_n
    g = tile // per_group
    first = g * group_m
    gs = min(tiles_m - first, group_m)
    local = tile - g * per_group
    tm = first + local % gs
    tn = local // gs
    if snake and (g & 1): tn = tiles_n - 1 - tn
    return tm, tn
def sim(n=8192, tile=256, ncl=74, group_m=8, cap_mb=110, kdir_alt=False, snake=False, order=None):
    tiles_m = tiles_n = n // tile
    kb_n = n // 64
    T = tiles_m * tiles_n
    blk = tile * 64 * 2
    cap = int(cap_mb * 2**20 / blk)
    lru = collections.OrderedDict()
    miss = 0
    waves = (T + ncl - 1) // ncl
    for w in range(waves):
        act = []
        for c in range(ncl):
            t = c + w * ncl
            if t < T: act.append(tile_coords(t, tiles_m, tiles_n, group_m, snake) if order is None else order[t])
        for s in range(kb_n):
            kb = (kb_n - 1 - s) if (kdir_alt and w % 2) else s
            for (tm, tn) in act:
                for key in (('A', tm, kb), ('B', kb, tn)):
                    if key in lru: lru.move_to_end(key)
                    else:
                        miss += 1; lru[key] = 1
                        if len(lru) > cap: lru.popitem(last=False)
    return miss * blk / 1e9
if __name__ == "__main__":
    for cap in (126, 100, 80, 60):
        for gm in (4, 6, 8, 10, 12, 16, 32):
            print(cap, gm, round(sim(group_m=gm, cap_mb=cap), 3), round(sim(group_m=gm, cap_mb=cap, kdir_alt=True), 3), flush=True)
