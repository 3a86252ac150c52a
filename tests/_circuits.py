"""Circuits shared by several GPU test modules (not a test module)."""
import numpy as np

from sv_inputs import Gate, haar_unitary, shift_x


def overlap_circuit(dims, seed, nranks):
    """Local gates on the low digits q_0..q_2 (controls on q_3.. below the top local qubit, which no
    gate touches) interleaved with Haar gates on the sharded qubits: every remap pairs a sharded
    qubit with the top local qubit and finds a pending local run it can overlap
    (SV_OPT_SHARD_OVERLAP)."""
    rng = np.random.default_rng(seed)
    n = len(dims)
    s = int(np.log2(nranks))
    top = n - s - 1
    gates = []
    for rep in range(6):
        for _ in range(5):
            t = int(rng.integers(0, 3))
            c = int(rng.integers(3, top))
            gates.append(Gate(t, (), (), haar_unitary(dims[t], rng)))
            gates.append(Gate(t, (c,), (1,), shift_x(dims[t], 1)))
        gates.append(Gate(n - 1 - rep % s, (), (), haar_unitary(2, rng)))
    return gates
