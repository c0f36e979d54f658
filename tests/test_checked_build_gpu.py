"""The checked build (make checked: device-side bounds and consistency checks
on every computed index, VXS_CHECKS; the analogue of the reference's
bounds-checked scalar backend, vec.hpp:85-120).  compute-sanitizer is not
available on this pool, so memory safety is established here: the small
parity subset (tools/sanitize_run.py, every key width, both orders, fallback,
argsort, partition, select, graph capture) runs clean against the checked
library and matches the oracle, and a deliberately inconsistent call (the
exchange pass run on different keys than the counting pass that filled its
workspace) is caught by a check instead of writing out of place."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(code_or_path, *, script=False, timeout=600):
    env = dict(os.environ, VXSORT_LIB="checked")
    cmd = [sys.executable, code_or_path] if script else [sys.executable, "-c", code_or_path]
    return subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, env=env, cwd=ROOT)


def test_parity_subset_runs_clean_under_checks(cuda):
    assert os.path.exists(os.path.join(ROOT, "paper_2205_05982_b200", "lib", "libvxsort_b200_checked.so"))
    r = _run(os.path.join(ROOT, "tools", "sanitize_run.py"), script=True)
    assert r.returncode == 0 and "ALL OK" in r.stdout, (r.returncode, r.stdout[-2000:], r.stderr[-2000:])
    assert "check failed" not in r.stdout


def test_inconsistent_exchange_is_caught(cuda):
    code = r'''
import sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_2205_05982_b200 as vx
assert vx.LIB_PATH.endswith("_checked.so")
rng = np.random.default_rng(1)
n = 300_000
a = torch.from_numpy(rng.integers(0, 2**63, n, dtype=np.uint64)).cuda()
b = torch.from_numpy(rng.integers(0, 2**63, n, dtype=np.uint64) >> np.uint64(20)).cuda()  # other keys
spl = torch.tensor([2**61, 2**62], dtype=torch.uint64).cuda()
ws = torch.empty(vx.workspace_bytes(n, "u64"), dtype=torch.uint8, device="cuda")
counts = vx.partition_counts(a, spl, ws)
out = torch.empty(n + 1024, dtype=torch.uint64, device="cuda")
addrs = torch.tensor([out.data_ptr()] * 3, dtype=torch.int64, device="cuda")
offs = torch.zeros(3, dtype=torch.int64, device="cuda")
try:
    vx.partition_exchange(b, 2, addrs, offs, ws)
    torch.cuda.synchronize()
except Exception as e:
    print("caught:", type(e).__name__)
    sys.exit(3)
print("not caught")
'''
    r = _run(code)
    assert r.returncode != 0, (r.stdout, r.stderr)
    assert "vxsort check failed" in r.stdout + r.stderr, (r.stdout[-2000:], r.stderr[-2000:])
