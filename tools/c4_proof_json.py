"""Writes tests/golden/c4_proof.json: C4's optimum (16) pinned with the
UNMODIFIED reference. "No 17" comes from tools/c4_split_proof.py — the
reference's own sequential solve() with a SharedBound floor on every piece of
a decomposition at the top of its search tree, one ledger line per piece
(tests/golden/c4_pieces.jsonl); "16 exists" from a 16-mapping found on the GPU
(gpurun_out/c4_witness.json, tools/gpu_call_r2_final.sh) that the reference's
oracle::verify accepts. Dev tool, dev container only.
usage: python tools/c4_proof_json.py [DEPTH=12]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import oracle as O  # noqa: E402
from c4_split_proof import decomposition  # noqa: E402

depth = int(sys.argv[1]) if len(sys.argv) > 1 else 12
tasks, removed = decomposition(depth)
ledger = [json.loads(l) for l in open(os.path.join(ROOT, "tests", "golden", "c4_pieces.jsonl")) if l.strip()]
by_tag = {p["piece"]: p for p in ledger}
missing = [t[0] for t in tasks if t[0] not in by_tag]
assert not missing, f"{len(missing)} pieces not run yet: {missing[:5]}"
pieces = [by_tag[t[0]] for t in tasks]
assert all(p["proved"] for p in pieces), [p for p in pieces if not p["proved"]]
wit = json.load(open(os.path.join(ROOT, "gpurun_out", "c4_witness.json")))
g, h = O.ref_random_graph(45, 0.5, 45000), O.ref_random_graph(45, 0.5, 45001)
pairs = [tuple(p) for p in wit["witness"]]
ok = O.ref_verify(g, h, pairs)
assert len(pairs) == 16 and ok == 1
out = {"instance": "ER n=45 p=0.5 seeds 45000/45001 (BASELINE.json configs[3])", "status": 0, "optimum": 16,
       "no_17": {"how": "tools/c4_split_proof.py: the reference's solve() with a SharedBound floor on each piece of "
                        "a decomposition at the top of its own search tree (branch v->u = the labelled pair G-v, "
                        "H-u with labels = adjacency to v, u, floor 15; v unmatched = G-v, H, decomposed again on "
                        "the next vertex; the last remainder floor 16); ledger tests/golden/c4_pieces.jsonl",
                 "depth": depth, "removed_vertices": removed, "pieces": len(pieces),
                 "max_piece_size": max(p["size"] for p in pieces),
                 "reference_nodes": sum(p["nodes"] for p in pieces),
                 "reference_cpu_seconds": round(sum(p["seconds"] for p in pieces), 1)},
       "witness": [list(p) for p in pairs], "witness_reference_verify": ok,
       "earlier_attempt": "reference solve_parallel (part_level 5, 7 threads) with a floor of 16: timeout after "
                          "6 h and 4.23e10 nodes (its tail ran on one thread)"}
json.dump(out, open(os.path.join(ROOT, "tests", "golden", "c4_proof.json"), "w"), indent=1)
print(json.dumps({k: v for k, v in out.items() if k != "witness"}))
