"""List registers and spill bytes per kernel from the ptxas -v logs of the libebs build
(paper_1911_03973_b200/csrc/build/*.ptxas.log).  Usage: python scripts/spills.py [--all]"""
import re
import subprocess
import sys
from pathlib import Path

BUILD = Path(__file__).resolve().parents[1] / "paper_1911_03973_b200" / "csrc" / "build"


def rows():
    for log in sorted(BUILD.glob("*.ptxas.log")):
        text = log.read_text()
        for b in re.split(r"ptxas info\s+: Compiling entry function '", text)[1:]:
            name = b.split("'")[0]
            sp = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", b)
            rg = re.search(r"Used (\d+) registers", b)
            dn = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
            yield (log.stem.split(".")[0], int(rg.group(1)) if rg else -1,
                   (int(sp.group(1)), int(sp.group(2))) if sp else (0, 0), dn)


if __name__ == "__main__":
    show_all = "--all" in sys.argv
    n_spill = 0
    for f, r, (st, ld), dn in rows():
        if show_all or st or ld:
            print(f"{f:10s} regs={r:3d} spill st/ld={st:4d}/{ld:4d}  {dn[:120]}")
        n_spill += bool(st or ld)
    print(f"kernels with spills: {n_spill}")
