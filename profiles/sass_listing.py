"""SASS of the hot kernels of libshapflow_b200.so (cuobjdump, no GPU needed).

    python profiles/sass_listing.py [outdir]

Writes <outdir>/sass_<kernel>.txt (full listing) and <outdir>/sass_census.md
(opcode counts per kernel, with the Blackwell markers: UTC*MMA = tcgen05.mma,
LDTM/STTM = tcgen05.ld/st, UBLKCP = cp.async.bulk, HMMA = legacy mma.sync).
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SO = os.path.join(ROOT, "paper_2506_22668_b200", "libshapflow_b200.so")
HOT = ["fused_tc_kernel", "isd_kernel", "tail_kernel", "floyd_kernel", "transpose_pairs_kernel",
       "transpose_tiles_kernel", "nib_forward_kernel", "nib_transpose_kernel", "list_forward_kernel",
       "list_transpose_kernel", "gram_tc_kernel", "chol_update_kernel", "assemble_pairs_kernel"]
MARKERS = ["UTCHMMA", "UTCQMMA", "UTCMMA", "UTCBAR", "LDTM", "STTM", "UBLKCP", "HMMA", "DFMA", "FFMA", "LDS", "ATOMS",
           "POPC", "SHFL"]


def main(outdir):
    os.makedirs(outdir, exist_ok=True)
    txt = subprocess.run(["cuobjdump", "-sass", SO], capture_output=True, text=True, check=True).stdout
    funcs = re.split(r"\n\s*Function : ", txt)
    census = collections.OrderedDict()
    for f in funcs[1:]:
        name = f.split("\n", 1)[0].strip()
        dem = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
        hit = next((h for h in HOT if h in dem), None)
        if not hit:
            continue
        key = dem.replace("(anonymous namespace)::", "").replace("<unnamed>::", "").replace("sfb::", "")
        key = re.sub(r"\(.*", "", key).replace("void ", "")
        ops = collections.Counter()
        for line in f.splitlines():
            m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
            if m:
                ops[m.group(1).split(".")[0]] += 1
        census[key] = ops
        safe = re.sub(r"[^A-Za-z0-9_]+", "_", key)[:80]
        with open(os.path.join(outdir, f"sass_{safe}.txt"), "w") as fo:
            fo.write(f"// {dem}\n// cuobjdump -sass {os.path.relpath(SO, ROOT)}\n")
            fo.write(f)
    with open(os.path.join(outdir, "sass_census.md"), "w") as fo:
        fo.write("# SASS opcode census of the hot kernels\n\n")
        fo.write("`python profiles/sass_listing.py` (cuobjdump -sass of libshapflow_b200.so, sm_100a). "
                 "UTC*MMA = tcgen05.mma, UTCBAR = tcgen05.commit, LDTM/STTM = tcgen05.ld/st, "
                 "UBLKCP = cp.async.bulk, HMMA = legacy mma.sync.\n\n")
        fo.write("| kernel | instructions | " + " | ".join(MARKERS) + " |\n")
        fo.write("|---|---:|" + "---:|" * len(MARKERS) + "\n")
        for k, ops in census.items():
            fo.write(f"| `{k}` | {sum(ops.values())} | " + " | ".join(str(ops.get(m, 0)) for m in MARKERS) + " |\n")
    print(open(os.path.join(outdir, "sass_census.md")).read())


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "round2", "sass"))
