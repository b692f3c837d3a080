"""GPU: the reference's own unit suites against the C++ drop-in.

oracle/_ref/conformance/shapflow_conformance is built here by
`make -C oracle conformance` (needs /root/reference; the binary travels to
the GPU box): proj/tests/test_sampler.cpp, test_gcn.cpp, test_solver.cpp and
test_pipeline.cpp, unchanged, compiled through the doctest shim in
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
    assert cases == 43 and failed == 0 and p.returncode == 0, out[-4000:]
