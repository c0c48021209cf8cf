import sys, hashlib, numpy as np
sys.path.insert(0, '.')
import paper_2103_14990_b200 as pb
for d, t in ((4, 20), (3, 20), (4, 10)):
    system = pb.build_chain_network(1000); spec = pb.make_benchmark_spec(system, t); mask = pb.build_locality_mask(system, d, t)
    from paper_2103_14990_b200.sls_core import build_column_classes_structural as bcs; cs = bcs(system, t, mask)
    op = pb.build_dynamics_operator(system, t); cg = pb.build_column_classes(op, mask)
    def hsh(cc):
        h = hashlib.blake2b(digest_size=8)
        for k in cc.classes:
            h.update(np.ascontiguousarray(k.g).tobytes()); h.update(np.ascontiguousarray(k.projector).tobytes())
        return h.hexdigest()
    print(d, t, 'structural', hsh(cs), 'general', hsh(cg), flush=True)
