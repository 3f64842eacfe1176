#!/usr/bin/env python3
"""Commits the SASS of the hot kernels as text (profiles/sass/*.sass) plus an
opcode summary (profiles/sass/SUMMARY.md): the north_star's "committed SASS
listing".  Reads the in-tree libsssp_cuda.so with cuobjdump -sass; no GPU.

    python tools/sass_dump.py
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2504_03667_b200", "libsssp_cuda.so")
OUT = os.path.join(ROOT, "profiles", "sass")

# (file stem, mangled-name regex, what it is)
KERNELS = [
    ("bucket_kernel_u8", r"_ZN9sssp_b20013bucket_kernelIhLb0EEEvNS_12BucketParamsE$",
     "bucket_kernel<u8, single solve> -- the default engine (config 3 headline)"),
    ("bucket_kernel_u8_multi", r"_ZN9sssp_b20013bucket_kernelIhLb1EEEvNS_12BucketParamsE$",
     "bucket_kernel<u8, MULTI> -- batched independent sources (config 5)"),
    ("cluster_scan_kernel_u8_16_4_packed",
     r"_ZN9sssp_b20019cluster_scan_kernelIhLi16ELi4ELb1ELb0ELb0EEEvNS_10ScanLaunchE$",
     "cluster_scan_kernel<u8, EPL 16, 4 warps, packed> -- the north-star n-round kernel (n=32768)"),
    ("dp_relax_kernel_u8", r"_ZN9sssp_b20015dp_relax_kernelIhEEvNS_8DpParamsE$",
     "dp_relax_kernel<u8> -- data-parallel relaxation rounds"),
    ("dp_tree_kernel_u8_fast", r"_ZN9sssp_b20014dp_tree_kernelIhLb0ELb1EEEvNS_8DpParamsE$",
     "dp_tree_kernel<u8, FAST> -- reconstruct_predecessors pass"),
    ("wide_scan_kernel", r"_ZN9sssp_b20016wide_scan_kernel",
     "wide_scan_kernel -- u64 weights/dist (kMaxWeight and n*max_w >= 2^32)"),
]

# opcodes worth pointing at (B200_PROFILING.md / blackwell guide mnemonics)
INTEREST = ["UBLKCP", "UTMALDG", "SYNCS", "LDGSTS", "LDGDEPBAR", "UCGABAR_ARV", "UCGABAR_WAIT",
            "CREDUX", "REDUX", "VIADDMNMX", "VIMNMX", "VIMNMX3", "PRMT", "SHFL", "ATOMS", "ATOMG",
            "ATOM", "RED", "REDG", "MEMBAR", "ERRBAR", "CCTL", "LDG", "LDS", "STS", "STG", "BAR",
            "VOTE", "POPC", "FLO", "BREV", "LDC", "S2UR", "UMOV", "CS2R"]


def functions(text):
    cur, buf = None, []
    for line in text.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            if cur:
                yield cur, "\n".join(buf)
            cur, buf = m.group(1), [line]
        elif cur:
            buf.append(line)
    if cur:
        yield cur, "\n".join(buf)


def opcodes(body):
    c = collections.Counter()
    for line in body.splitlines():
        m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
        if m:
            c[m.group(2)] += 1
    return c


def main():
    os.makedirs(OUT, exist_ok=True)
    text = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True,
                          check=True).stdout
    funcs = dict(functions(text))
    rows = []
    for stem, pat, what in KERNELS:
        names = [f for f in funcs if re.search(pat, f)]
        if not names:
            print(f"missing: {stem}", file=sys.stderr)
            continue
        name = names[0]
        body = funcs[name]
        with open(os.path.join(OUT, stem + ".sass"), "w") as f:
            f.write(f"// {what}\n// cuobjdump -sass paper_2504_03667_b200/libsssp_cuda.so, {name}\n")
            f.write(body + "\n")
        c = opcodes(body)
        rows.append((stem, what, sum(c.values()), c))
    with open(os.path.join(OUT, "SUMMARY.md"), "w") as f:
        f.write("# SASS opcode summary (sm_100a, `tools/sass_dump.py`)\n\n")
        f.write("Counts are static instructions in the listing (not executed counts).\n\n")
        for stem, what, tot, c in rows:
            f.write(f"## {stem}.sass\n\n{what}; {tot} instructions.\n\n")
            hits = [(k, c[k]) for k in INTEREST if c.get(k)]
            f.write("| opcode | count |\n|---|---|\n")
            for k, v in hits:
                f.write(f"| {k} | {v} |\n")
            top = ", ".join(f"{k} {v}" for k, v in c.most_common(12))
            f.write(f"\nTop opcodes: {top}\n\n")
    print(f"wrote {len(rows)} listings to {OUT}")


if __name__ == "__main__":
    main()
