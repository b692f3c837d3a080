"""TEST INFRASTRUCTURE ONLY (conformance build, oracle/Makefile `conformance`).

Marks the reference's definitions of the hot-path API functions WEAK in a
compiled reference object, so that the B200 drop-in's strong definitions
(paper_2506_22668_b200/dropin/shapflow_dropin.cpp) replace them at link time
while every other function of that translation unit (model / mask I/O,
assemble_problem, explain_nodes, select_nodes, ...) stays the reference's.
This is what a maintainer does by deleting those bodies from sampler.cpp /
gcn.cpp / solver.cpp / explain.cpp."""
import subprocess
import sys

HOT = ["plan_sizes", "generate_masks", "predict_probs", "predict", "predict_batched", "solve_cgls",
       "solve_direct", "rank_edges", "explain_node", "auto_samples", "node_sampling_seed"]


def main(obj):
    out = subprocess.run(["nm", "--defined-only", "-g", obj], check=True, capture_output=True, text=True).stdout
    syms = [ln.split()[-1] for ln in out.splitlines() if ln.split() and ln.split()[-2] in ("T", "W")]
    dem = subprocess.run(["c++filt"], input="\n".join(syms), check=True, capture_output=True, text=True).stdout
    weak = []
    for mangled, d in zip(syms, dem.splitlines()):
        for h in HOT:
            if d.startswith(f"shapflow::{h}("):
                weak.append(mangled)
    if weak:
        subprocess.run(["objcopy"] + [f"--weaken-symbol={s}" for s in weak] + [obj], check=True)
    print(f"{obj}: weakened {len(weak)} hot-path definitions")


if __name__ == "__main__":
    for o in sys.argv[1:]:
        main(o)
