"""profiles/traffic.json from a round's `ncu --set full` summaries
(tools/ncu_summary.py output, profiles/TAG_ncu_*.txt): DRAM read + write
bytes per launch of each bench kernel label, for bench.py's
roofline.traffic.

    python tools/make_traffic.py TAG
"""
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
# bench.py kernel label -> (summary file suffix, kernel name regex)
LABELS = {
    "resize_down": ("resize", r"resize_down2_tma_kernel<3>"),
    "resize_up": ("resize", r"resize_up2_kernel<3>"),
    "resize_normalize_chw": ("fused", r"resize_strip_kernel<unsigned char, 3, 2(, 0)?>"),
    "warp_affine": ("affine", r"warp_affine_src_kernel<float, 3>"),
    "warp_perspective": ("persp", r"warp_persp_tile_kernel<3>"),
    "gray_u8 32-frame batch (one launch)": ("graybatch", r"gray_u8_vec_kernel"),
    "gray_u8 per frame (graph of 32 launches)": ("gray", r"gray_u8_flat_kernel<8>"),
}


def parse(path):
    out, cur = [], None
    units = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    for line in open(path):
        if line.startswith("== "):
            cur = {"name": line[3:].strip()}
            out.append(cur)
        elif cur is not None and "dram__bytes_" in line:
            m = re.match(r"\s*dram__bytes_(read|write)\.sum = ([0-9.]+) (\w+)", line)
            if m:
                cur[m.group(1)] = float(m.group(2)) * units[m.group(3)]
    return out


def main(tag):
    res = {}
    for label, (suffix, rx) in LABELS.items():
        path = os.path.join(ROOT, "profiles", f"{tag}_ncu_{suffix}.txt")
        if not os.path.exists(path):
            continue
        ks = [k for k in parse(path) if re.search(rx, k["name"]) and "read" in k]
        if not ks:
            continue
        k = ks[0]
        res[label] = {"dram_bytes": int(k["read"] + k.get("write", 0)), "kernel": k["name"][:80],
                      "source": f"profiles/{tag}_ncu_{suffix}.txt (ncu --set full, cold caches)"}
    with open(os.path.join(ROOT, "profiles", "traffic.json"), "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r02a")
