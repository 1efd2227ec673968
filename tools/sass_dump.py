"""Regenerate profiles/sass/*.sass (the SASS of every hot-path kernel in
libnvc.so) and profiles/r2_sass_evidence.txt (instruction counts and the
tcgen05 / TMEM / bulk-copy mnemonics).  Usage: sass_dump.py [libnvc.so]"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_2506_05930_b200", "libnvc.so")
HOT = ["k_enc_tiles2", "k_mlp_ts", "k_mlp_tiles", "k_nls32g", "k_ndi32", "k_adam_bulk", "k_adam_mlp", "k_train3",
       "k_train_tc", "k_tr_encode", "k_tr_scatter", "k_reduce_parts", "k_targets_sorted", "k_screen_round0",
       "k_screen_finish", "k_morton_order", "k_world", "k_shade", "k_cluster_tgt", "k_cluster_draws", "k_cs_step2",
       "k_gbuffer", "k_factors", "k_ris_initial", "k_restir_temporal", "k_restir_spatial"]
MNEM = ["UTCHMMA", "UTCBAR", "LDTM", "STTM", "UTCCP", "UBLKCP", "UTMALDG", "ELECT", "REDUX", "FHFMA", "IMAD.WIDE",
        "DFMA", "DADD", "RED.E.ADD"]
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
funcs = re.split(r"\n\s+Function : ", sass)[1:]
out_dir = os.path.join(ROOT, "profiles", "sass")
os.makedirs(out_dir, exist_ok=True)
for f in os.listdir(out_dir):
    if f.endswith(".sass"):
        os.remove(os.path.join(out_dir, f))
rows = []
for f in funcs:
    mangled = f.split("\n", 1)[0].strip()
    dem = subprocess.run(["c++filt", mangled], capture_output=True, text=True).stdout.strip()
    m = re.search(r"(k_\w+)(<[^>(]*>)?\(", dem)
    if not m or m.group(1) not in HOT:
        continue
    name = m.group(1) + (("_" + re.sub(r"[^0-9a-zA-Z]+", "_", m.group(2)).strip("_")) if m.group(2) else "")
    ops = re.findall(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_]+(?:\.[A-Z0-9_]+)*)", f)
    with open(os.path.join(out_dir, name + ".sass"), "w") as fh:
        fh.write(f"// {dem}\n// cuobjdump -sass {os.path.basename(lib)}\n" + f)
    c = collections.Counter()
    for op in ops:
        for k in MNEM:
            if op == k or op.startswith(k + "."):
                c[k] += 1
    rows.append((name, len(ops), c))
with open(os.path.join(ROOT, "profiles", "r2_sass_evidence.txt"), "w") as fh:
    fh.write("SASS of the hot kernels in libnvc.so (cuobjdump -sass; tools/sass_dump.py): instruction count and\n"
             "the mnemonics that show tcgen05 MMA (UTCHMMA), its commit (UTCBAR), TMEM loads/stores (LDTM/STTM),\n"
             "bulk async copies (UBLKCP), mixed-precision FMA (FHFMA), 64-bit integer multiply (IMAD.WIDE), FP64\n\n")
    for name, n, c in sorted(rows):
        fh.write(f"{name:34s} {n:6d} instr  " + "  ".join(f"{v:3d} {k}" for k, v in sorted(c.items())) + "\n")
print(open(os.path.join(ROOT, "profiles", "r2_sass_evidence.txt")).read())
