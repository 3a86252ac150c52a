import sys, time, subprocess; sys.path.insert(0,'.')
def run(nr, nq, k, block, tmo=40):
    code = f"""
import sys; sys.path.insert(0,'.')
import paper_2410_17876_b200 as P
from sv_inputs import config_circuit
dims, gates = config_circuit(4, nqubits={nq})
st = P.State.loopback(dims, {nr}) if {nr} > 1 else P.State(dims)
st.apply_circuit(gates[:{k}], fuse=True, check=False, block={block})
st.sync(); print('ok')
"""
    try:
        r = subprocess.run([sys.executable, '-c', code], timeout=tmo, capture_output=True, text=True)
        return 'ok' in r.stdout
    except subprocess.TimeoutExpired:
        return False
for rep in range(3):
    print('P2 nq7 full block', run(2, 7, 300, True), flush=True)
print('P2 nq7 full noblock', run(2, 7, 300, False), flush=True)
lo, hi = 0, 300
while hi - lo > 1:
    mid = (lo + hi) // 2
    ok = run(2, 7, mid, True)
    print(mid, ok, flush=True)
    if ok: lo = mid
    else: hi = mid
print('first failing prefix', hi, flush=True)
