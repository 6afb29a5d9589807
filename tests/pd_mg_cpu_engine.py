"""CPU engine for the sharded multigrid schedule (paper_2006_12883_b200.mg_sharded):
vectors are torch CPU float64 tensors (so gloo can move them), operators scipy
CSR, the block-Jacobi ILU(0) and dense LU the oracle's restatements of the
reference (oracle/paradiff_oracle.py).  Test infrastructure only."""

import numpy as np
import scipy.sparse as sp
import torch

from oracle import paradiff_oracle as O


class CpuEngine:
    def operator(self, A):
        return sp.csr_matrix(A)

    def preconditioner(self, A_own, nblocks, grid=None, m=0):
        A_own = O.canon(A_own)
        return O.OBlockJacobi(A_own, nblocks) if nblocks > 1 else O.OIlu0(A_own)

    def coarse_solver(self, A):
        return O.ODenseLU(O.canon(A))

    def vec(self, a):
        return torch.as_tensor(np.asarray(a, dtype=np.float64)).clone()

    def zeros(self, n):
        return torch.zeros(int(n), dtype=torch.float64)

    def empty(self, n):
        return torch.empty(int(n), dtype=torch.float64)

    def apply(self, op, x):
        return torch.from_numpy(op @ x.numpy())

    def residual(self, op, b, x):
        return torch.from_numpy(b.numpy() - op @ x.numpy())

    def precond(self, pre, v):
        return torch.from_numpy(np.asarray(pre.solve(v.numpy()), dtype=np.float64))

    def coarse(self, lu, b):
        return torch.from_numpy(np.asarray(lu.solve(b.numpy()), dtype=np.float64))

    def dot(self, a, b):
        return float(np.dot(a.numpy(), b.numpy()))

    def size(self, a):
        return int(a.numel())

    def cat(self, a, b):
        return torch.cat([a, b])

    def slice_tail(self, x, k):
        return x[x.numel() - k:].clone()

    def host(self, x):
        return x.numpy()

    def comm_tensor(self, x):
        return x
