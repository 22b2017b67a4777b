"""Memory accounting of the implicit method.

For every BASELINE config: the complex words the paper counts for the
implicit method and for explicit padding, and what this implementation
holds -- the user's input arrays plus the device workspace the C ABI asks
for (idc_workspace_bytes) -- and, when a comparison run has been recorded
(tools/cufft_explicit.py --out profiles/r01_cufft_compare.json), the bytes the
explicit cuFFT convolution actually allocated on the B200.

Paper formulas (complex words per convolution):
  cconv1d   4m both ways ("storage requirements ... identical")
  hconv1d   2(floor(N/2)+1) = 3m+2 both ways, m = 2c, N = 3m
  tconv1d   6(m+1) implicit, 3(2m+1) explicit
  cconv2d   4 mx my + 2 my implicit, 8 mx my explicit
  hconv2d   2(2mx-1)my + 2(mx+1)my + 2(my/2+1) = 6 mx my + my + 2 implicit,
            9 mx my - 6 my explicit minimum
  tconv2d   6*2mx(my+1) + 3(my+1) = 12 mx my + 12 mx + 3 my + 3 implicit,
            3*4mx(2my+1) = 24 mx my + 12 mx explicit
  cconv3d   4 mx my mz + 2 my mz + 2 mz implicit, 16 mx my mz explicit
            
  hconv3d   6mx(2my-1)mz + 2(my+1)mz + 2(mz/2+1) implicit (the itemised
            count; the paper's printed closed form is 2mz short, AMB-21),
            27 mx my mz explicit

    python tools/memory_report.py [--compare profiles/r01_cufft_compare.json] [--out profiles/r01_memory.md]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

WORD = 16  # bytes per complex128 word


def paper_words(kind, mx, my=1, mz=1):
    """(implicit, explicit) complex words of ONE convolution, as the paper
    counts them (formulas in the module docstring)."""
    if kind == "cconv1d":
        return 4 * mx, 4 * mx
    if kind == "hconv1d":
        return 3 * mx + 2, 3 * mx + 2
    if kind == "tconv1d":
        return 6 * (mx + 1), 3 * (2 * mx + 1)
    if kind == "cconv2d":
        return 4 * mx * my + 2 * my, 8 * mx * my
    if kind == "hconv2d":
        return 2 * (2 * mx - 1) * my + 2 * (mx + 1) * my + 2 * (my // 2 + 1), 9 * mx * my - 6 * my
    if kind == "tconv2d":
        return 6 * 2 * mx * (my + 1) + 3 * (my + 1), 3 * 4 * mx * (2 * my + 1)
    if kind == "cconv3d":
        return 4 * mx * my * mz + 2 * my * mz + 2 * mz, 16 * mx * my * mz
    if kind == "hconv3d":
        return (6 * mx * (2 * my - 1) * mz + 2 * (my + 1) * mz + 2 * (mz // 2 + 1), 27 * mx * my * mz)
    raise ValueError(kind)


def input_words(kind, mx, my=1, mz=1):
    """Words of the user's input arrays in this implementation's layouts
    (include/idconv.h), one convolution."""
    return {"cconv1d": 2 * mx, "hconv1d": 2 * mx, "tconv1d": 3 * mx, "cconv2d": 2 * mx * my,
            "hconv2d": 2 * (2 * mx - 1) * my, "tconv2d": 3 * 2 * mx * my, "cconv3d": 2 * mx * my * mz,
            "hconv3d": 2 * (2 * mx - 1) * (2 * my - 1) * mz}[kind]


# (config, kind, sizes (mx, my, mz), batch) -- BASELINE.json configs
CONFIGS = [
    ("c1", "cconv1d", (1024, 1, 1), 32768),
    ("c2a", "hconv1d", (4096, 1, 1), 4096),
    ("c2b", "tconv1d", (4096, 1, 1), 4096),
    ("c3a", "cconv2d", (1024, 1024, 1), 1),
    ("c3b", "cconv2d", (256, 256, 1), 64),
    ("c4", "hconv2d", (2048, 2048, 1), 1),
    ("c4t", "tconv2d", (2048, 2048, 1), 1),
    ("c5a", "cconv3d", (512, 512, 512), 1),
    ("c5b", "hconv3d", (512, 512, 512), 1),
]


def ours_words(kind, sizes, batch):
    """(input words, workspace words) of this implementation for the config."""
    from paper_1008_1366_b200 import idconv
    code = getattr(idconv, kind.upper())
    mx, my, mz = sizes
    dims = {1: (mx,), 2: (mx, my), 3: (mx, my, mz)}[1 if kind.endswith("1d") else (2 if kind.endswith("2d") else 3)]
    ws = idconv.workspace_bytes(code, *dims, batch=batch if kind in ("cconv1d", "hconv1d", "tconv1d", "cconv2d") else 1)
    return input_words(kind, mx, my, mz) * batch, ws // WORD


def report(compare=None):
    measured = {}
    if compare and os.path.exists(compare):
        for r in json.load(open(compare)):
            measured[r["config"]] = r
    rows = []
    for name, kind, sizes, batch in CONFIGS:
        imp, exp = (w * batch for w in paper_words(kind, *sizes))
        inp, ws = ours_words(kind, sizes, batch)
        m = measured.get(name, {})
        ex_meas = None
        if m.get("explicit_extra_bytes") is not None:
            ex_meas = m["input_bytes"] // WORD + m["explicit_extra_bytes"] // WORD
        rows.append(dict(config=name, kind=kind, sizes=list(sizes), batch=batch, paper_implicit_words=imp,
                         paper_explicit_words=exp, ours_input_words=inp, ours_workspace_words=ws,
                         ours_total_words=inp + ws, explicit_cufft_measured_words=ex_meas,
                         explicit_error=m.get("error")))
    return rows


def markdown(rows):
    gb = lambda w: f"{w * WORD / 1e9:.3g}" if w is not None else "—"
    out = ["| config | problem | paper implicit (GB) | paper explicit (GB) | ours: inputs + workspace (GB) | "
           "ours / paper implicit | explicit cuFFT measured (GB) |", "|---|---|---|---|---|---|---|"]
    for r in rows:
        meas = gb(r["explicit_cufft_measured_words"]) if r["explicit_cufft_measured_words"] else (
            "OOM" if r["explicit_error"] else "—")
        out.append(f"| {r['config']} | {r['kind']} {tuple(s for s in r['sizes'] if s > 1)} x{r['batch']} | "
                   f"{gb(r['paper_implicit_words'])} | {gb(r['paper_explicit_words'])} | "
                   f"{gb(r['ours_input_words'])} + {gb(r['ours_workspace_words'])} | "
                   f"{r['ours_total_words'] / r['paper_implicit_words']:.3f} | {meas} |")
    return "\n".join(out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--compare", default=os.path.join(ROOT, "profiles", "r01_cufft_compare.json"))
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    rows = report(a.compare)
    md = markdown(rows)
    print(md)
    if a.out:
        with open(a.out, "w") as fh:
            fh.write(md + "\n")
        with open(os.path.splitext(a.out)[0] + ".json", "w") as fh:
            json.dump(rows, fh, indent=1)


if __name__ == "__main__":
    main()
