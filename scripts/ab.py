"""A/B runner (experiments): time prebuilt library variants with the same
bench section, alternating, on one box.

  python scripts/ab.py --rounds 3 --section hash build/ab/lib_x.so default ...

`default` = the in-tree libvsb200.so.  Variants are built here (CPU) with
  python scripts/ab.py --build NAME DEF1=1 DEF2=0 ...
which writes build/ab/lib_NAME.so.
"""

from __future__ import annotations

import argparse
import json
import os
import pathlib
import subprocess
import sys

ROOT = pathlib.Path(__file__).resolve().parent.parent
SECTIONS = {
    "hash": ["--no-cpu", "--no-mc", "--no-stream", "--no-rc", "--no-e2e", "--no-server", "--steps", "200"],
    "mc": ["--no-cpu", "--no-stream", "--no-rc", "--no-e2e", "--no-server", "--steps", "5", "--mc-steps", "20",
           "--no-mc-parity"],
    "stream": ["--no-cpu", "--no-mc", "--no-rc", "--no-e2e", "--no-server", "--steps", "5"],
    "server": ["--no-cpu", "--no-mc", "--no-rc", "--no-e2e", "--no-stream", "--steps", "5"],
    "rc": ["--no-cpu", "--no-mc", "--no-stream", "--no-e2e", "--no-server", "--steps", "5"],
    "config1": ["--no-cpu", "--no-mc", "--no-stream", "--no-rc", "--no-e2e", "--no-server", "--steps", "3"],
}


def pick(d: dict, section: str):
    if section == "hash":
        return {"value": round(d["value"]), "kernel_ms": round(d["roofline"]["kernel_ms"], 4),
                "ms_per_step": round(d["ms_per_step"], 4), "ok": d["parity_ok"]}
    if section == "config1":
        c = d.get("config1") or {}
        return {"hash_M_ops": round(c.get("hash", {}).get("value", 0)), "ms": c.get("hash", {}).get("ms_per_step"),
                "mc_blocks": c.get("mc", {}).get("value"), "ok": c.get("ok"), "error": c.get("error")}
    s = d.get(section) or {}
    out = {k: s.get(k) for k in ("value", "ms_per_step", "ms_per_tick", "ok", "error") if k in s}
    if "roofline" in s:
        out["kernel_ms"] = s["roofline"].get("kernel_ms")
        out["frac"] = s["roofline"].get("frac")
    for k in ("tick_only", "server_tick", "compact", "incremental_packs"):
        if k in s:
            out[k] = s[k].get("ms_per_step") if isinstance(s[k], dict) else s[k]
    return out


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "--build":
        name, defs = sys.argv[2], tuple(sys.argv[3:])
        sys.path.insert(0, str(ROOT))
        from paper_1805_03709_b200 import build

        out = ROOT / "build" / "ab" / f"lib_{name}.so"
        out.parent.mkdir(parents=True, exist_ok=True)
        print(build.build(out=out, defines=defs))
        return
    p = argparse.ArgumentParser()
    p.add_argument("--rounds", type=int, default=2)
    p.add_argument("--section", default="hash")
    p.add_argument("--extra", default="")
    p.add_argument("libs", nargs="+")
    a = p.parse_args()
    for r in range(a.rounds):
        for lib in a.libs:
            env = dict(os.environ)
            if lib != "default":
                env["VSB_LIB"] = str(ROOT / lib)
            cmd = [sys.executable, str(ROOT / "bench.py"), *SECTIONS[a.section], *a.extra.split()]
            res = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=900)
            try:
                d = json.loads(res.stdout.strip().splitlines()[-1])
                print(r, lib, json.dumps(pick(d, a.section)), flush=True)
            except Exception:  # noqa: BLE001
                print(r, lib, "FAILED", res.stderr[-800:], flush=True)


if __name__ == "__main__":
    main()
