import sys, json, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import numpy as np
from paper_2512_11112_b200 import artifacts as A, runtime as rt
m = json.load(open('tests/golden/fuzz/expected.json'))['f41']
vals = {k: np.array(v, np.uint32) for k, v in m['inputs'].items()}
g = A.read_circuit_file('tests/golden/fuzz/f41.mpcg').to_graph(vals)
for n in (2, 3):
    rep = rt.run_local(g, n, vals, dealer_seed=9)
    print(n, rep.outputs.tolist(), rep.output_digest, rep.scalar_triples_consumed)
print('expected', m)
for i, n in enumerate(g.nodes): print(i, n.kind, n.lanes, n.operands, n.is_private, n.const_val, n.name)
print(g.const_inputs)
