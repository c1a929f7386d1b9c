"""Negative control of the peer-protocol self-test: with libebs built with
-DEBS_PEER_BREAK_PARITY=1 (one halo slot, no double buffering) the concurrent self-test must
report wrong values; with the product library it reports none.
  make -C paper_1911_03973_b200/csrc BUILD=build_brk OUT=../variants/libebs_break_parity.so \
       EXTRA=-DEBS_PEER_BREAK_PARITY=1
  EBS_LIB_PATH=paper_1911_03973_b200/variants/libebs_break_parity.so EBS_PEER_TIMEOUT=5 \
       python scripts/peer_selftest_control.py"""
import os
import sys

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_1911_03973_b200 import dist  # noqa: E402
from paper_1911_03973_b200._lib import LIB_PATH  # noqa: E402
from paper_1911_03973_b200.inputs import config_problem  # noqa: E402

for cfg, size, P in ((4, 7, 2), (4, 7, 5), (5, 8, 8)):
    pr = config_problem(cfg, seed=1, size=size)
    m = pr["mesh"]
    prob, _ = dist.emulate(pr["batch"], m.n_nodes, pr["dirichlet"], P, peer=True)
    n = prob.comm.selftest(300)
    try:
        prob.comm.status()
        st = "ok"
    except Exception as e:  # noqa: BLE001
        st = f"error word set ({e})"[:80]
    print(f"{os.path.basename(LIB_PATH)}: C{cfg} size {size} P={P}: {n} wrong values, status {st}",
          flush=True)
    prob.comm.close()
