import sys, subprocess; sys.path.insert(0,'.')
def run(code, tmo=30):
    try:
        r = subprocess.run([sys.executable, '-c', code], timeout=tmo, capture_output=True, text=True)
        return 'ok' in r.stdout, r.stderr[-200:]
    except subprocess.TimeoutExpired:
        return False, 'timeout'
base = """
import sys; sys.path.insert(0,'.')
import paper_2410_17876_b200 as P
from sv_inputs import config_circuit, Gate
dims, gates = config_circuit(4, nqubits=7)
ldims = dims[:18]
g = {{i: gates[i] for i in range(300)}}
sel = {sel}
st = P.State(ldims)
{opts}
st.apply_circuit([g[i] for i in sel], fuse=True, check=False, block=True)
st.sync(); print('ok')
"""
cases = {
 'run170_181': list(range(170, 182)),
 'pair179_181': [179, 181],
 'only179': [179],
 'only181': [181],
}
for name, sel in cases.items():
    for opts in ["", "st.set_option(P.sv.SV_OPT_PASS_GROUPS, 1)", "st.set_option(P.sv.SV_OPT_PASS_THREADS, 256)"]:
        print(name, opts, run(base.format(sel=sel, opts=opts)), flush=True)
