"""compute-sanitizer over small invocations of every kernel family:
memcheck and initcheck must be clean; racecheck may report only the
shared-memory hazards DESIGN.md section 11 documents as benign (the in-place
pointer doubling / chase of k_tile, where every value a thread can observe is
a later vertex of the same ascending path).  Reports go to gpurun_out/ when
EG_SANITIZER_LOG is set (summaries are committed under profiles/)."""
import os
import re
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CASES = ["c1", "t64", "d5", "knn"]
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
# kernels whose shared-memory hazards are the documented benign ones
BENIGN_RACE_KERNELS = ("k_tile",)


def _run(tool, case):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    # every kernel is instrumented: initcheck must see the writes of the cub
    # scans / sorts the library calls, or it reports their outputs as
    # uninitialized when our kernels read them
    cmd = [SAN, f"--tool={tool}", "--print-limit", "200"]
    if tool == "racecheck":
        cmd += ["--racecheck-report", "hazard"]
    cmd += [sys.executable, os.path.join(ROOT, "tools", "sanitize_case.py"), case]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1200, cwd=ROOT)
    out = r.stdout + r.stderr
    if "closed on this pool" in out:
        # the GPU pool's operators replaced compute-sanitizer with a stub (runs under
        # it left GPUs needing a reset); the clean reports of earlier runs are under
        # profiles/r02/sanitizer/
        pytest.skip("compute-sanitizer is disabled on this GPU pool")
    d = os.environ.get("EG_SANITIZER_LOG")
    if d:
        os.makedirs(d, exist_ok=True)
        with open(os.path.join(d, f"sanitizer_{tool}_{case}.txt"), "w") as fh:
            fh.write(out)
    assert f"sanitize case {case}: ok" in out, out[-3000:]
    return out


@pytest.mark.parametrize("case", CASES)
def test_memcheck(case):
    out = _run("memcheck", case)
    assert "ERROR SUMMARY: 0 errors" in out, out[-3000:]


@pytest.mark.parametrize("case", CASES)
def test_initcheck(case):
    out = _run("initcheck", case)
    assert "ERROR SUMMARY: 0 errors" in out, out[-3000:]


def _benign_lines():
    """k_grid3d.cu lines marked `benign-race`: the in-place pointer doubling
    and chase of the tile kernel."""
    src = os.path.join(ROOT, "paper_2303_02724_b200", "csrc", "k_grid3d.cu")
    return {i + 1 for i, ln in enumerate(open(src)) if "benign-race" in ln}


@pytest.mark.parametrize("case", CASES)
def test_racecheck(case):
    out = _run("racecheck", case)
    m = re.search(r"RACECHECK SUMMARY: (\d+) hazard", out)
    if m is None or int(m.group(1)) == 0:
        return
    # every access of every reported hazard must be on a documented benign line
    acc = re.findall(r"(?:Read|Write) Thread \([^)]*\) at (?:void )?(?:eg::)?(\w+).* in ([\w.]+):(\d+)", out)
    assert acc, out[-3000:]
    ok = _benign_lines()
    bad = sorted({(k, f, int(n)) for k, f, n in acc if not (k in BENIGN_RACE_KERNELS and f == "k_grid3d.cu"
                                                             and int(n) in ok)})
    assert not bad, f"undocumented shared-memory races at {bad}:\n{out[-3000:]}"
