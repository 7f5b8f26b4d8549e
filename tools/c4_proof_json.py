"""Writes tests/golden/c4_proof.json: C4's optimum (16) pinned with the
UNMODIFIED reference. "No 17" comes from tools/c4_split_proof.py — the
reference's own sequential solve() with a SharedBound floor on every piece of
a decomposition at the top of its search tree (gpurun_out/c4_split_proof.json;
optionally the remainder piece proved by a deeper decomposition,
gpurun_out/c4_split_proof_skip5.json); "16 exists" from a 16-mapping found on
the GPU (gpurun_out/c4_witness.json) that the reference's oracle::verify
accepts. Dev tool, dev container only."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402

OUT = os.path.join(ROOT, "gpurun_out")
main = json.load(open(os.path.join(OUT, "c4_split_proof.json")))
pieces = list(main["pieces"])
deeper = os.path.join(OUT, "c4_split_proof_skip5.json")
remainder = [p for p in pieces if p["piece"].startswith("unmatched")]
assert len(remainder) == 1
if not remainder[0]["proved"] and os.path.exists(deeper):  # the remainder, decomposed further
    d = json.load(open(deeper))
    assert d["all_proved"], "the deeper decomposition did not prove the remainder"
    pieces = [p for p in pieces if not p["piece"].startswith("unmatched")] + d["pieces"]
assert all(p["proved"] for p in pieces), [p for p in pieces if not p["proved"]]
wit = json.load(open(os.path.join(OUT, "c4_witness.json")))
g, h = O.ref_random_graph(45, 0.5, 45000), O.ref_random_graph(45, 0.5, 45001)
pairs = [tuple(p) for p in wit["witness"]]
ok = O.ref_verify(g, h, pairs)
assert len(pairs) == 16 and ok == 1
out = {"instance": "ER n=45 p=0.5 seeds 45000/45001 (BASELINE.json configs[3])", "status": 0, "optimum": 16,
       "no_17": {"how": "tools/c4_split_proof.py: the reference's solve() with a SharedBound floor on each piece of "
                        "a decomposition at the top of its own search tree (branch v->u = the labelled pair G-v, "
                        "H-u with labels = adjacency to v, u, floor 15; v unmatched = G-v, H, decomposed again; "
                        "the last remainder floor 16)",
                 "removed_vertices": main["removed_vertices"], "pieces": len(pieces),
                 "reference_nodes": sum(p["nodes"] for p in pieces),
                 "reference_cpu_seconds": round(sum(p["seconds"] for p in pieces), 1)},
       "witness": [list(p) for p in pairs], "witness_reference_verify": ok,
       "earlier_attempt": "reference solve_parallel (part_level 5, 7 threads) with a floor of 16: timeout after "
                          "6 h and 4.23e10 nodes (its tail ran on one thread)"}
json.dump(out, open(os.path.join(ROOT, "tests", "golden", "c4_proof.json"), "w"), indent=1)
print(json.dumps({k: v for k, v in out.items() if k != "witness"}))
