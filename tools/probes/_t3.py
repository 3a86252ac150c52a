import sys, time; sys.path.insert(0,'.')
import paper_2410_17876_b200 as P
from sv_inputs import config_circuit
seq = [int(x) for x in sys.argv[1].split(',')]
nq = int(sys.argv[2]); block = sys.argv[3] == '1'
dims, gates = config_circuit(4, nqubits=nq)
ga = P.sv._GateArray(gates)
for nr in seq:
    st = P.State(dims) if nr == 1 else P.State.loopback(dims, nr)
    t = time.time()
    st.apply_circuit(ga, fuse=True, check=False, block=block)
    st.sync(); print(nr, 'apply', round(time.time() - t, 3), flush=True)
    st.close()
print('done', flush=True)
