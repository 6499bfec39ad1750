import sys, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from conftest import load_case, index_from_case
import paper_2301_06672_b200 as pkg
k, P, prec, name = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], sys.argv[4]
c = load_case(name); idx = index_from_case(c)
try:
    lists, ns = pkg.search_batch(idx, c["queries"], pkg.SearchParams(k=k, nprobe=P, precision=prec))
    from oracle import c_oracle
    ids, d, n2 = c_oracle.search_batch(c["coarse"], c["centers"], c["list_off"], c["ids"], c["codes"], c["queries"], k, P, prec)
    print(name, k, P, prec, "OK", np.array_equal(lists.ids, ids), np.array_equal(lists.distances, d))
except Exception as e:
    print(name, k, P, prec, "ERR", str(e)[:150])
