"""CPU engine for timeslab.run_windows built on the oracle (TEST INFRASTRUCTURE ONLY).

Lets the sharded PFASST schedule (paper_2006_12883_b200/timeslab.py) run under
torch.distributed/gloo on CPU: the per-worker numerics come from the oracle's
restatement of pfasst.py, communication buffers are CPU torch tensors.
"""

import numpy as np
import torch

from oracle import paradiff_oracle as O
from paper_2006_12883_b200.errors import SolverError
from paper_2006_12883_b200.timeslab import worker_range


def _guard(fn):
    def wrapped(*a, **k):
        try:
            return fn(*a, **k)
        except O.OracleSolverError as exc:
            raise SolverError(str(exc)) from exc
    return wrapped


class OracleEngine:
    def __init__(self, levels, trs, nu, u_init, Nt, P, rank, size):
        self.lv, self.trs, self.nu = levels, trs, nu
        self.L = len(levels)
        self.w0, self.w1 = worker_range(P, rank, size)
        self.W = self.w1 - self.w0
        S, M = levels[0].mh.size, levels[0].M
        self.out = np.zeros((Nt, M, S))
        self.u_start = np.asarray(u_init, dtype=np.float64).copy()
        self.nrecv = max(self.L - 1, 1)
        f64 = torch.float64
        self.halo_in = [torch.zeros(levels[l].mh.size, dtype=f64) for l in range(self.nrecv)]
        self.halo_out = [torch.zeros(levels[l].mh.size, dtype=f64) for l in range(self.nrecv)]
        self.c_in = torch.zeros(levels[-1].mh.size, dtype=f64)
        self.c_out = torch.zeros(levels[-1].mh.size, dtype=f64)
        self.fine_term = torch.zeros(S, dtype=f64)
        self.msgs = None

    num_levels = property(lambda self: self.L)
    local_workers = property(lambda self: self.W)

    def setup_window(self, start):
        self.chain = [self.u_start]
        for tr in self.trs:
            self.chain.append(tr.down_u0(self.chain[-1]))
        self.st = [[[np.tile(self.chain[l], (lev.M, 1)), self.chain[l].copy(), None]
                    for l, lev in enumerate(self.lv)] for _ in range(self.W)]
        r = self.lv[0].res_norm(*self.st[0][0])
        self._r0 = r
        return np.full(self.W, r)

    def window_r0(self):
        return self._r0

    def halo_buffers(self):
        return self.halo_in

    def halo_out_buffers(self):
        return self.halo_out

    def receive(self, halo):
        for l in range(self.nrecv):
            for w in range(1, self.W):
                self.st[w][l][1] = self.msgs[l][w - 1].copy()
            if halo is not None:
                self.st[0][l][1] = halo[l].numpy().copy()

    @_guard
    def fine_sweeps(self):
        for w in range(self.W):
            for _ in range(self.nu):
                self.st[w][0][0] = self.lv[0].sweep(*self.st[w][0])

    @_guard
    def coarse_down(self):
        for w in range(self.W):
            s = self.st[w]
            for l in range(1, self.L):
                tr = self.trs[l - 1]
                RU = tr.down(s[l - 1][0])
                tau = O.fas_tau(self.lv[l - 1], self.lv[l], tr, s[l - 1][0], s[l - 1][2])
                s[l] = [RU, s[l][1], tau]
                if l < self.L - 1:
                    for _ in range(self.nu):
                        s[l][0] = self.lv[l].sweep(*s[l])

    def coarse_start_buffer(self):
        return self.c_in

    def load_coarse_start(self, buf):
        buf.copy_(torch.from_numpy(self.chain[-1].copy()))

    @_guard
    def coarse_chain(self, u0c):
        L = self.L
        for w in range(self.W):
            self.st[w][L - 1][1] = (u0c.numpy().copy() if w == 0
                                    else self.st[w - 1][L - 1][0][-1].copy())
            for _ in range(self.nu):
                self.st[w][L - 1][0] = self.lv[L - 1].sweep(*self.st[w][L - 1])
        self.c_out.copy_(torch.from_numpy(self.st[self.W - 1][L - 1][0][-1].copy()))
        return self.c_out

    def coarse_last_buffer(self):
        return self.c_out

    @_guard
    def coarse_up(self):
        for w in range(self.W):
            s = self.st[w]
            for l in range(self.L - 2, -1, -1):
                tr = self.trs[l]
                RU = tr.down(s[l][0])
                s[l][0] = s[l][0] + tr.up(s[l + 1][0] - RU)
                if 0 < l < self.L - 1:
                    for _ in range(self.nu):
                        s[l][0] = self.lv[l].sweep(*s[l])

    def publish(self):
        self.msgs = [[self.st[w][l][0][-1].copy() for w in range(self.W)]
                     for l in range(self.nrecv)]
        for l in range(self.nrecv):
            self.halo_out[l].copy_(torch.from_numpy(self.msgs[l][self.W - 1]))
        return np.array([self.lv[0].res_norm(*self.st[w][0]) for w in range(self.W)])

    def store_window(self, start):
        for w in range(self.W):
            self.out[start + self.w0 + w] = self.st[w][0][0]

    def last_fine_terminal(self):
        self.fine_term.copy_(torch.from_numpy(self.st[self.W - 1][0][0][-1].copy()))
        return self.fine_term

    def set_window_start(self, t):
        self.u_start = t.numpy().copy()
