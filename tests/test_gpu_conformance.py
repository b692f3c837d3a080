"""GPU: the reference's own unit suites against the C++ drop-in.

oracle/_ref/conformance/shapflow_conformance is built here by
`make -C oracle conformance` (needs /root/reference; the binary travels to
the GPU box): proj/tests/test_sampler.cpp, test_gcn.cpp, test_solver.cpp,
test_pipeline.cpp, test_fidelity.cpp, test_oracle.cpp and test_document.cpp,
unchanged, compiled through the doctest shim in
tests/conformance/ and linked so that plan_sizes, generate_masks,
predict_probs, predict, predict_batched, solve_cgls, solve_direct,
rank_edges, explain_node, auto_samples and node_sampling_seed come from
paper_2506_22668_b200/dropin/shapflow_dropin.cpp (libshapflow_b200 on the
GPU) and everything else from the reference core.
"""
import os
import re
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "conformance", "shapflow_conformance")


def test_reference_suites_pass_on_the_dropin():
    if not os.path.exists(BIN):
        pytest.skip("conformance binary not built (needs /root/reference at build time)")
    env = dict(os.environ, SHAPFLOW_B200_DEVICE="0")
    p = subprocess.run([BIN], capture_output=True, text=True, timeout=900, env=env)
    out = p.stdout + p.stderr
    print(out[-6000:])
    m = re.search(r"test cases: (\d+) \| (\d+) passed \| (\d+) failed", out)
    assert m, out[-2000:]
    cases, passed, failed = map(int, m.groups())
    assert cases == 65 and failed == 0 and p.returncode == 0, out[-4000:]


ACC = os.path.join(ROOT, "oracle", "_ref", "conformance", "shapflow_acceptance")


@pytest.mark.slow
def test_reference_acceptance_criteria_on_the_dropin():
    """proj/tests/acceptance.cpp (the reference's 11 acceptance criteria) over
    the drop-in, against the same program over the unmodified reference core
    (tests/golden/acceptance_reference.txt, `make -C oracle acceptance_ref`):
    every criterion the reference passes must pass. Criterion 10 measures the
    CPU implementation's thread scaling (p = 1, 2, 4 host threads, prediction
    time dominant) and does not apply to the device path; criteria 6 (needs
    the reference CLI binary, not buildable here) and 8 (efficiency gap
    6.2e-3 > 1e-3 on its own systems) fail in the reference itself."""
    if not os.path.exists(ACC):
        pytest.skip("acceptance binary not built (needs /root/reference at build time)")
    env = dict(os.environ, SHAPFLOW_B200_DEVICE="0")
    p = subprocess.run([ACC], capture_output=True, text=True, timeout=1800, env=env)
    out = p.stdout + p.stderr
    print(out[-8000:])

    def verdicts(text):
        got = {}
        for ln in text.splitlines():
            m = re.match(r"(PASS|FAIL) criterion (\d+):", ln)  # acceptance.cpp:61-65
            if m:
                got[int(m.group(2))] = m.group(1)
        return got

    ours = verdicts(out)
    ref = verdicts(open(os.path.join(ROOT, "tests", "golden", "acceptance_reference.txt")).read())
    assert len(ours) == 11 and len(ref) == 11, out[-3000:]
    regressions = [c for c in sorted(ref) if ref[c] == "PASS" and ours[c] != "PASS" and c != 10]
    assert not regressions, out[-4000:]
