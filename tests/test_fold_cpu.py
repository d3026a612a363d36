"""CPU: the parity-split half matrices the plan uploads (etd_setup_fold_matrices)
reproduce the dense eigenbasis transform exactly in exact arithmetic and to
rounding in FP64, for odd and even n and both storage layouts.

The identity: the DST-I eigenbasis P(i,k) = c sin((i+1)(k+1)pi/(n+1))
(operators.cpp:43-53) has P(n-1-i, k) = (-1)^k P(i, k), so with s_i = g_i + g_{n-1-i},
d_i = g_i - g_{n-1-i} (i < h = (n+1)/2) the forward transform is
ghat_{2q} = sum_i P(i,2q) s_i and ghat_{2q+1} = sum_i P(i,2q+1) d_i, and the
backward one is g_i = o_i + e_i, g_{n-1-i} = o_i - e_i with o, e the even / odd
mode sums.  This file restates the kernels' index maps (etd_kernels.cuh FOLD) in
numpy on top of the library's matrices."""
import ctypes as C

import numpy as np
import pytest

import paper_2601_06849_b200 as etd
from oracle import Oracle


def fold_mats(n, mode):
    h = (n + 1) // 2
    ld = (h + 15) // 16 * 16 if mode == 0 else 2 * h
    size = 2 * h * ld if mode == 0 else h * ld
    ff, fb = np.zeros(size), np.zeros(size)
    rc = etd.lib().etd_setup_fold_matrices(n, mode, ff.ctypes.data_as(C.c_void_p), fb.ctypes.data_as(C.c_void_p))
    assert rc == 0
    if mode == 0:
        return ff.reshape(2 * h, ld)[:, :h], fb.reshape(2 * h, ld)[:, :h]
    return ff.reshape(h, 2 * h).T, fb.reshape(h, 2 * h).T   # -> [row][col]


def parity_major(n):
    h = (n + 1) // 2
    return [2 * q for q in range(h)] + [2 * q + 1 for q in range(n - h)]


def fold_forward(g, FF, n):
    """FOLD 1/3/4: rows r of the interleaved matrix -> parity-major positions."""
    h = (n + 1) // 2
    i = np.arange(h)
    s = g[..., i] + g[..., n - 1 - i]
    d = g[..., i] - g[..., n - 1 - i]
    out = np.zeros(g.shape[:-1] + (n,))
    for r in range(2 * h):
        grp, pos = (r >> 3) & 1, (r >> 4) * 8 + (r & 7) + ((r >> 3) & 1) * h
        if pos < n:
            out[..., pos] = (d if grp else s) @ FF[r]
    return out


def fold_backward(gh, FB, n):
    """FOLD 2: even / odd mode groups -> o, e -> g_i = o + e, g_{n-1-i} = o - e."""
    h = (n + 1) // 2
    S = gh[..., :h]
    A = np.concatenate([gh[..., h:], np.zeros(gh.shape[:-1] + (2 * h - n,))], -1)
    out = np.zeros(gh.shape[:-1] + (n,))
    for r in range(0, 2 * h, 16):
        for t in range(8):
            io = (r >> 4) * 8 + t
            if io < h:
                o, e = S @ FB[r + t], A @ FB[r + 8 + t]
                out[..., io] = o + e
                out[..., n - 1 - io] = o - e
    return out


@pytest.mark.parametrize("n", [15, 16, 31, 47, 48, 63, 127, 255])
@pytest.mark.parametrize("mode", [0, 1])
def test_fold_matrices_reproduce_dense_transform(n, mode):
    FF, FB = fold_mats(n, mode)
    P, _ = Oracle.spectral_factor(n, 2.0, -1.0)   # the reference P (column-major flattening)
    P = np.asarray(P).reshape(n, n).T if np.asarray(P).ndim == 1 else np.asarray(P)
    g = np.random.default_rng(n).uniform(-1, 1, (5, n))
    perm = parity_major(n)
    dense_fwd = g @ P                          # ghat_k = sum_i P(i,k) g_i
    assert np.max(np.abs(fold_forward(g, FF, n) - dense_fwd[:, perm])) <= 1e-13 * n
    gh = np.random.default_rng(n + 1).uniform(-1, 1, (5, n))   # parity-major modes
    nat = np.zeros_like(gh)
    nat[:, perm] = gh
    assert np.max(np.abs(fold_backward(gh, FB, n) - nat @ P.T)) <= 1e-13 * n


def test_fold_centre_entries_exact():
    """Odd n: the centre column of the even forward group is P/2 (s counts the
    centre twice), the odd group's centre entries are exactly 0 (so the centre
    output is o + 0 = o - 0 bitwise)."""
    n = 31
    h = 16
    FF, FB = fold_mats(n, 0)
    P, _ = Oracle.spectral_factor(n, 2.0, -1.0)
    P = np.asarray(P).reshape(n, n).T if np.asarray(P).ndim == 1 else np.asarray(P)
    for r in range(2 * h):
        grp, q = (r >> 3) & 1, (r >> 4) * 8 + (r & 7)
        if grp == 0:
            assert FF[r, h - 1] == 0.5 * P[h - 1, 2 * q]
        else:
            assert FF[r, h - 1] == 0.0
            if q == h - 1:
                assert np.all(FB[r] == 0.0)


def test_fold_matrices_refuse_unfoldable_n():
    buf = np.zeros(4096)
    p = buf.ctypes.data_as(C.c_void_p)
    assert etd.lib().etd_setup_fold_matrices(25, 0, p, p) != 0   # h = 13
    assert etd.lib().etd_setup_fold_matrices(31, 2, p, p) != 0   # bad layout


# ---------------------------------------------------------------- second level
def fold2_mats(n, mode):
    h = (n + 1) // 2
    H = h // 2
    ldH = (H + 15) // 16 * 16 if mode == 0 else 2 * H
    ldh = (h + 15) // 16 * 16 if mode == 0 else 2 * h
    ga = np.zeros(2 * H * ldH if mode == 0 else H * ldH)
    gb, go, ge = np.zeros_like(ga), np.zeros_like(ga), np.zeros_like(ga)
    fb = np.zeros(2 * h * ldh if mode == 0 else h * ldh)
    vp = lambda a: a.ctypes.data_as(C.c_void_p)
    assert etd.lib().etd_setup_fold2_matrices(n, mode, vp(ga), vp(gb), vp(fb), vp(go), vp(ge)) == 0
    if mode == 0:
        small = lambda a: a.reshape(2 * H, ldH)[:, :H]
        return small(ga), small(gb), fb.reshape(2 * h, ldh)[:, :h], small(go), small(ge)
    small = lambda a: a.reshape(H, 2 * H).T
    return small(ga), small(gb), fb.reshape(h, 2 * h).T, small(go), small(ge)


def fold2_modes(n):
    """mode of each level-2 position: p < h -> 2p; h + c -> 4c + 1 (c < H), 4(c - H) + 3."""
    h = (n + 1) // 2
    H = h // 2
    return [2 * p for p in range(h)] + [4 * c + 1 for c in range(H)] + [4 * c + 3 for c in range(H - 1)]


def fold2_stack(g, n, from1=False):
    """etd_fold2 restated: [s even i | s odd i | d_k + d_{2H-2-k} | d_k - d_{2H-2-k}]."""
    h = (n + 1) // 2
    H = h // 2
    if from1:
        s, d = g[..., :h], g[..., h:]
    else:
        i = np.arange(h)
        s = g[..., i] + g[..., n - 1 - i]
        d = (g[..., i] - g[..., n - 1 - i])[..., :h - 1]
    k = np.arange(H)
    c = 2 * H - 2 - k
    dd_s = d[..., k] + d[..., c]
    dd_d = (d[..., k] - d[..., c])[..., :H - 1]
    return np.concatenate([s[..., 0::2], s[..., 1::2], dd_s, dd_d], -1)


def fold2_forward(st, GA, GB, n):
    """FOLD 5 (GA: boxes [0,H), [H,2H); +/- to positions q, h-1-q) and FOLD 4 (GB: boxes
    [2H,3H), [3H,4H-1); positions 2H + 8b + t%8 + group H)."""
    h = (n + 1) // 2
    H = h // 2
    out = np.zeros(st.shape[:-1] + (n,))
    A0, A1 = st[..., :H], st[..., H:2 * H]
    B0 = st[..., 2 * H:3 * H]
    B1 = np.concatenate([st[..., 3 * H:], np.zeros(st.shape[:-1] + (1,))], -1)
    for r in range(0, 2 * H, 16):
        for t in range(8):
            q = (r >> 4) * 8 + t
            if q < H:
                a, b = A0 @ GA[r + t], A1 @ GA[r + 8 + t]
                out[..., q] = a + b
                out[..., h - 1 - q] = a - b
    for r in range(2 * H):
        grp = (r >> 3) & 1
        pos = 2 * H + (r >> 4) * 8 + (r & 7) + grp * H
        if pos < n:
            out[..., pos] = (B1 if grp else B0) @ GB[r]
    return out


@pytest.mark.parametrize("n", [31, 63, 127, 255, 511])
@pytest.mark.parametrize("mode", [0, 1])
def test_fold2_reproduces_dense_transform(n, mode):
    GA, GB, FB2, GO, GE = fold2_mats(n, mode)
    P, _ = Oracle.spectral_factor(n, 2.0, -1.0)
    P = np.asarray(P).reshape(n, n).T if np.asarray(P).ndim == 1 else np.asarray(P)
    modes = fold2_modes(n)
    assert sorted(modes) == list(range(n))
    rng = np.random.default_rng(n)
    g = rng.uniform(-1, 1, (5, n))
    dense_fwd = g @ P
    got = fold2_forward(fold2_stack(g, n), GA, GB, n)
    assert np.max(np.abs(got - dense_fwd[:, modes])) <= 1e-13 * n
    # the x corrector's input: x_back_src writes the first-level stack of f(What)
    h = (n + 1) // 2
    i = np.arange(h)
    first = np.concatenate([g[:, i] + g[:, n - 1 - i], (g[:, i] - g[:, n - 1 - i])[:, :h - 1]], -1)
    got1 = fold2_forward(fold2_stack(first, n, from1=True), GA, GB, n)
    assert np.max(np.abs(got1 - dense_fwd[:, modes])) <= 1e-13 * n
    # backward: the first-level FOLD 2 kernel reading level-2 positions
    gh = rng.uniform(-1, 1, (5, n))          # level-2 positions
    nat = np.zeros_like(gh)
    nat[:, modes] = gh
    assert np.max(np.abs(fold_backward(gh, FB2, n) - nat @ P.T)) <= 1e-13 * n


def test_fold2_matrices_reject_ineligible_sizes():
    p = C.c_void_p(0)
    assert etd.lib().etd_setup_fold2_matrices(47, 0, p, p, p, p, p) != 0   # h = 24: H not a multiple of 8
    assert etd.lib().etd_setup_fold2_matrices(64, 0, p, p, p, p, p) != 0   # even n


def fold2_backward(gh, GO, GE, n):
    """Level-2 backward restated: (sigma, delta) of the even-mode pairs (q, h-1-q) (the
    FOLD 5 forward epilogue stores them, sd_out); FOLD 4 over them with GO -> o at even /
    odd i; FOLD 2 over the odd-mode group with GE -> e, e mirrored about its centre;
    etd_unfold2: g_i = o_i + e_i, g_{n-1-i} = o_i - e_i."""
    h = (n + 1) // 2
    H = h // 2
    q = np.arange(H)
    sig = gh[..., q] + gh[..., h - 1 - q]
    dlt = gh[..., q] - gh[..., h - 1 - q]
    mid = np.zeros(gh.shape[:-1] + (n,))               # [o even i | o odd i | e]
    for r in range(2 * H):                           # FOLD 4 launch, kbase = nbase = 0
        grp = (r >> 3) & 1
        pos = (r >> 4) * 8 + (r & 7) + grp * H
        if pos < 2 * H:
            mid[..., pos] = (dlt if grp else sig) @ GO[r]
    B0 = gh[..., 2 * H:3 * H]
    B1 = np.concatenate([gh[..., 3 * H:], np.zeros(gh.shape[:-1] + (1,))], -1)
    m = 2 * H - 1
    for r in range(0, 2 * H, 16):                    # FOLD 2 launch, kbase = nbase = 2H, n_axis = 2H - 1
        for t in range(8):
            io = (r >> 4) * 8 + t
            if io < H:
                o, e = B0 @ GE[r + t], B1 @ GE[r + 8 + t]
                mid[..., 2 * H + io] = o + e
                mid[..., 2 * H + m - 1 - io] = o - e
    spos = lambda i: H + i // 2 if i % 2 else i // 2
    out = np.zeros_like(mid)
    for i in range(h):
        o = mid[..., spos(i)]
        if i == h - 1:
            out[..., i] = o
        else:
            e = mid[..., 2 * H + i]
            out[..., i] = o + e
            out[..., n - 1 - i] = o - e
    return out


@pytest.mark.parametrize("n", [31, 63, 127, 255, 511])
@pytest.mark.parametrize("mode", [0, 1])
def test_fold2_backward_reproduces_dense_transform(n, mode):
    _, _, _, GO, GE = fold2_mats(n, mode)
    P, _ = Oracle.spectral_factor(n, 2.0, -1.0)
    P = np.asarray(P).reshape(n, n).T if np.asarray(P).ndim == 1 else np.asarray(P)
    modes = fold2_modes(n)
    gh = np.random.default_rng(n + 3).uniform(-1, 1, (5, n))   # level-2 positions
    nat = np.zeros_like(gh)
    nat[:, modes] = gh
    assert np.max(np.abs(fold2_backward(gh, GO, GE, n) - nat @ P.T)) <= 1e-13 * n


# ---------------------------------------------------------------- fused level-2 backward
def back6_mat(n, mode):
    H = (n + 1) // 4
    R = (4 * H + 63) // 64 * 64                    # whole (par 0, par 1) block pairs
    ld = (H + 15) // 16 * 16 if mode == 0 else R
    g6 = np.zeros(R * ld if mode == 0 else H * ld)
    assert etd.lib().etd_setup_back6_matrix(n, mode, g6.ctypes.data_as(C.c_void_p)) == 0
    return g6.reshape(R, ld)[:, :H] if mode == 0 else g6.reshape(H, R).T


def back6_backward(st, G6, n):
    """etd_back6 restated: the input stack [sigma | delta | Y_lo | Y_hi] (4 boxes of H
    along the axis), B rows in 32-row blocks (parity b & 1, orbit base b >> 1) of four
    fragments (o_k, o_c', eo_k, ee_k), fragment A box = parity for types 0/1, else the
    type; the orbit epilogue e = eo +- ee, g = o +- e at k, n-1-k, c', n-1-c'."""
    H = (n + 1) // 4
    boxes = [st[..., q * H:(q + 1) * H] for q in range(3)]
    boxes.append(np.concatenate([st[..., 3 * H:], np.zeros(st.shape[:-1] + (1,))], -1))
    acc = {}
    for r in range(G6.shape[0]):
        blk, t = r >> 5, (r >> 3) & 3
        par, kb = blk & 1, blk >> 1
        k = 16 * kb + 2 * (r & 7) + par
        if k >= H:
            assert not G6[r].any()
            continue
        box = par if t < 2 else t
        acc[(k, t)] = boxes[box] @ G6[r]
    out = np.zeros(st.shape[:-1] + (n,))
    for k in range(H):
        O1, O2, EO, EE = (acc[(k, t)] for t in range(4))
        ek, ec = EO + EE, EO - EE
        out[..., k] = O1 + ek
        out[..., n - 1 - k] = O1 - ek
        if k == H - 1:
            out[..., 2 * H - 1] = O2            # the centre o_{2H-1}
        else:
            c = 2 * H - 2 - k
            out[..., c] = O2 + ec
            out[..., n - 1 - c] = O2 - ec
    return out


@pytest.mark.parametrize("n", [31, 63, 127, 255, 511, 1023])
@pytest.mark.parametrize("mode", [0, 1])
def test_back6_equals_two_launch_backward_bitwise(n, mode):
    """G6 holds exactly GO's and GE's entries, regrouped: every accumulator is the
    same dot product of the same vectors, so the fused backward equals the round-1
    two-launch + unfold path bit for bit, and the dense transform to rounding."""
    _, _, _, GO, GE = fold2_mats(n, mode)
    G6 = back6_mat(n, mode)
    h = (n + 1) // 2
    H = h // 2
    gh = np.random.default_rng(n + 11).uniform(-1, 1, (4, n))   # level-2 positions
    q = np.arange(H)
    st = np.concatenate([gh[:, q] + gh[:, h - 1 - q], gh[:, q] - gh[:, h - 1 - q], gh[:, 2 * H:]], -1)
    got = back6_backward(st, G6, n)
    assert np.max(np.abs(got - fold2_backward(gh, GO, GE, n))) <= 1e-15 * n
    # bitwise: every G6 row is the GO / GE row of the same output
    for r in range(G6.shape[0]):
        blk, t = r >> 5, (r >> 3) & 3
        k = 16 * (blk >> 1) + 2 * (r & 7) + (blk & 1)
        if k >= H:
            continue
        if t < 2:
            i = k if t == 0 else (2 * H - 1 if k == H - 1 else 2 * H - 2 - k)
            ro = ((i >> 1) >> 3) * 16 + (i & 1) * 8 + ((i >> 1) & 7)   # GO row of output i = 2q + group
            assert np.array_equal(G6[r], GO[ro])
        else:
            ro = (k >> 3) * 16 + (t - 2) * 8 + (k & 7)                   # GE row of (k, group t - 2)
            assert np.array_equal(G6[r], GE[ro])
    P, _ = Oracle.spectral_factor(n, 2.0, -1.0)
    P = np.asarray(P).reshape(n, n).T if np.asarray(P).ndim == 1 else np.asarray(P)
    nat = np.zeros_like(gh)
    nat[:, fold2_modes(n)] = gh
    assert np.max(np.abs(got - nat @ P.T)) <= 1e-13 * n
    # the centre row of ee and its last column are exact zeros (odd group: 2H - 1 modes)
    for r in range(G6.shape[0]):
        blk, t = r >> 5, (r >> 3) & 3
        k = 16 * (blk >> 1) + 2 * (r & 7) + (blk & 1)
        if t == 3 and k < H:
            assert G6[r, H - 1] == 0.0 and (k != H - 1 or not G6[r].any())


def test_back6_matrix_rejects_ineligible_sizes():
    p = C.c_void_p(0)
    assert etd.lib().etd_setup_back6_matrix(47, 0, p) != 0
    assert etd.lib().etd_setup_back6_matrix(64, 1, p) != 0
