"""SASS listings + mnemonic census of the shipped kernels (cuobjdump -sass of the built
libgemm_f16.so), evidence that the path runs on tcgen05 / TMEM / TMA:
UTCHMMA (tcgen05.mma kind::f16), LDTM (tcgen05.ld), UTMALDG (TMA load), UTMAREDG (TMA
reduce-add store), UTMASTG (TMA store), UTCBAR (tcgen05.commit), SYNCS (mbarrier).
usage: python tools/sass_census.py OUTDIR"""
import collections, os, re, subprocess, sys
ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
LIB = os.path.join(ROOT, "paper_2108_13191_b200", "libgemm_f16.so")
SHIPPED = {   # file stem -> mangled-name fragment
    "sass_pair_256x256_k128_f32_reduce": "KCfgILi2ELi256ELi3ELb0ELi1ELi128ELb0ELi1ELb1EEELb0EE",
    "sass_pair_256x256_k128_f32_reduce_streamk": "KCfgILi2ELi256ELi3ELb0ELi1ELi128ELb0ELi1ELb1EEELb1EE",
    "sass_pair_256x512_f16_wide": "gemm_f16_sm100_wide_kernelINS_4WCfgILi4EEELb0EE",
    # (selectable, not picked: the B-multicast kernel behind MCB and MCH)
    "sass_pair2_256x256_mc_f32": "KCfgILi2ELi256ELi3ELb0ELi1ELi128ELb0ELi2ELb1EEELb0EE",
}
KEYS = ["UTCHMMA", "UTCQMMA", "UTCBAR", "LDTM", "STTM", "UTMALDG", "UTMAREDG", "UTMASTG", "UTMAPF", "UBLKCP",
        "SYNCS", "ELECT", "STS", "LDS", "BAR", "HMMA"]
out = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "r02")
os.makedirs(out, exist_ok=True)
sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
funcs = re.split(r"\n\s*Function : ", sass)[1:]
census = []
for f in funcs:
    name = f.split("\n", 1)[0].strip()
    ops = collections.Counter()
    for line in f.split("\n"):
        m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
        if m:
            ops[m.group(1)] += 1
            ops[m.group(1) + (m.group(2) or "")] += 0
    census.append((name, ops, f))
    for stem, frag in SHIPPED.items():
        if frag in name:
            with open(os.path.join(out, stem + ".txt"), "w") as fh:
                fh.write(f"// cuobjdump -sass {os.path.relpath(LIB, ROOT)}\n// Function : {name}\n{f}")
with open(os.path.join(out, "sass_census.txt"), "w") as fh:
    fh.write("# cuobjdump -sass paper_2108_13191_b200/libgemm_f16.so: mnemonic counts per kernel\n")
    fh.write("# kernel | " + " ".join(KEYS) + "\n")
    for name, ops, _ in census:
        fh.write(name + " | " + " ".join(f"{k}={ops[k]}" for k in KEYS) + "\n")
    # full variant forms of the tcgen05 / TMA ops in the shipped kernels
    for name, ops, f in census:
        if any(frag in name for frag in SHIPPED.values()):
            forms = sorted(set(re.findall(r"\b(UTC\w+(?:\.\w+)*|LDTM(?:\.\w+)*|UTMA\w+(?:\.\w+)*)", f)))
            fh.write(f"\n## {name}\n" + "\n".join(forms) + "\n")
print(open(os.path.join(out, "sass_census.txt")).read()[:3000])
