"""Writes tests/golden/gen_hashes.json (generator drift detector).  Calls only
sdnngen (structure), never the CUDA path.  Run: python tests/golden/make_gen_hashes.py"""
import hashlib
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import sdnngen as g  # noqa: E402
from test_gen import SPECS  # noqa: E402

out = {name: g.structure_hash(mk()) for name, mk in SPECS.items()}
rp, idx = g.ms_inputs(1024, 1000)
out["ms_1024_1000"] = hashlib.sha256(rp.tobytes() + idx.tobytes()).hexdigest()
json.dump(out, open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "gen_hashes.json"), "w"), indent=1)
print(out)
