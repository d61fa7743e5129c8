"""Pins for the oracle's fp64 cell equations and evaluators — CPU only.

The paper only cites the cells; the readings (SURVEY App. A / DESIGN.md §3) are pinned here
against library routines on special cases that reduce to them (torch.nn.LSTMCell, GRUCell,
RNNCell, LSTM), closed forms, and agreement of two independently written evaluators.
"""
import numpy as np
import pytest
import torch

import workloads as W
from oracle import cells
from oracle.evaluate import evaluate_levels, evaluate_recursive

torch.set_default_dtype(torch.float64)


def _rand(gen, *shape, s=0.5):
    return gen.uniform(-s, s, size=shape)


def test_treelstm_leaf_equals_lstmcell_with_zero_state():
    gen = np.random.default_rng(0)
    h = 6
    p = {"W": _rand(gen, 3 * h, h), "b": _rand(gen, 3 * h)}
    x = _rand(gen, h)
    cell = torch.nn.LSTMCell(h, h)
    Wi, Wo, Wu = p["W"][:h], p["W"][h:2 * h], p["W"][2 * h:]
    bi, bo, bu = p["b"][:h], p["b"][h:2 * h], p["b"][2 * h:]
    with torch.no_grad():  # torch gate order [i, f, g, o]
        cell.weight_ih.copy_(torch.tensor(np.concatenate([Wi, np.zeros((h, h)), Wu, Wo])))
        cell.bias_ih.copy_(torch.tensor(np.concatenate([bi, np.zeros(h), bu, bo])))
        cell.weight_hh.zero_(); cell.bias_hh.zero_()
        ht, ct = cell(torch.tensor(x)[None], (torch.zeros(1, h), torch.zeros(1, h)))
    hh, cc = cells.treelstm_leaf(p, x)
    np.testing.assert_allclose(hh, ht[0].numpy(), rtol=0, atol=1e-14)
    np.testing.assert_allclose(cc, ct[0].numpy(), rtol=0, atol=1e-14)


def test_treelstm_internal_with_zero_right_child_equals_lstmcell():
    """U^r = 0 (right child has h_r = 0, c_r = 0): internal = LSTMCell(0, (h_l, c_l))."""
    gen = np.random.default_rng(1)
    h = 5
    p = {"W": _rand(gen, 5 * h, 2 * h), "b": _rand(gen, 5 * h)}
    hl, cl = _rand(gen, h), _rand(gen, h)
    hh, cc = cells.treelstm_internal(p, hl, cl, np.zeros(h), np.zeros(h))
    U = p["W"][:, :h]
    Ui, Ufl, Uo, Uu = U[:h], U[h:2 * h], U[3 * h:4 * h], U[4 * h:]
    b = p["b"]
    cell = torch.nn.LSTMCell(h, h)
    with torch.no_grad():
        cell.weight_ih.zero_(); cell.bias_ih.zero_()
        cell.weight_hh.copy_(torch.tensor(np.concatenate([Ui, Ufl, Uu, Uo])))
        cell.bias_hh.copy_(torch.tensor(np.concatenate([b[:h], b[h:2 * h], b[4 * h:], b[3 * h:4 * h]])))
        ht, ct = cell(torch.zeros(1, h), (torch.tensor(hl)[None], torch.tensor(cl)[None]))
    np.testing.assert_allclose(hh, ht[0].numpy(), atol=1e-14)
    np.testing.assert_allclose(cc, ct[0].numpy(), atol=1e-14)


def test_treelstm_internal_right_slot_is_used():
    """Guards a dropped f_r / c_r term: swapping children changes the result unless symmetric."""
    gen = np.random.default_rng(2)
    h = 4
    p = {"W": _rand(gen, 5 * h, 2 * h), "b": _rand(gen, 5 * h)}
    a = [_rand(gen, h) for _ in range(4)]
    h1, c1 = cells.treelstm_internal(p, a[0], a[1], a[2], a[3])
    h2, c2 = cells.treelstm_internal(p, a[0], a[1], a[2], a[3] + 1.0)
    assert np.all(np.abs(c2 - c1) > 0)
    sig_fr = 1 / (1 + np.exp(-(p["W"][2 * h:3 * h] @ np.concatenate([a[0], a[2]]) + p["b"][2 * h:3 * h])))
    np.testing.assert_allclose(c2 - c1, sig_fr, atol=1e-14)   # dc/dc_r = s(f_r), exactly linear


def test_treegru_leaf_equals_grucell_zero_state():
    gen = np.random.default_rng(3)
    h = 5
    p = {"W": _rand(gen, 2 * h, h), "b": _rand(gen, 2 * h)}
    x = _rand(gen, h)
    cell = torch.nn.GRUCell(h, h)
    with torch.no_grad():  # torch gate order [r, z, n]; n = tanh(W_in x + b_in + r*(W_hn h + b_hn))
        cell.weight_ih.copy_(torch.tensor(np.concatenate([np.zeros((h, h)), p["W"][:h], p["W"][h:]])))
        cell.bias_ih.copy_(torch.tensor(np.concatenate([np.zeros(h), p["b"][:h], p["b"][h:]])))
        cell.weight_hh.zero_(); cell.bias_hh.zero_()
        ht = cell(torch.tensor(x)[None], torch.zeros(1, h))
    np.testing.assert_allclose(cells.treegru_leaf(p, x), ht[0].numpy(), atol=1e-14)


def test_treegru_internal_spine_equals_grucell():
    """h_r = 0 and U_{.r} = 0: internal = GRUCell(0, h_l) (linear-before-reset reading)."""
    gen = np.random.default_rng(4)
    h = 4
    W = _rand(gen, 5 * h, 2 * h)
    W[3 * h:4 * h, h:] = 0; W[4 * h:, :h] = 0
    b = _rand(gen, 5 * h)
    b[2 * h:3 * h] = 0  # r_r bias irrelevant once a_r = 0 ... keep general below
    p = {"W": W, "b": b}
    hl = _rand(gen, h)
    # a_r = U_nr*0 + b_nr must vanish for the reduction: zero b_nr
    p["b"][4 * h:] = 0
    out = cells.treegru_internal(p, hl, np.zeros(h))
    cell = torch.nn.GRUCell(h, h)
    with torch.no_grad():  # h' = (1-z) n + z h ; n = tanh(r*(W_hn h + b_hn)); r = s(W_hr h + b_hr)
        cell.weight_ih.zero_(); cell.bias_ih.zero_()
        cell.weight_hh.copy_(torch.tensor(np.concatenate([W[h:2 * h, :h], W[:h, :h], W[3 * h:4 * h, :h]])))
        cell.bias_hh.copy_(torch.tensor(np.concatenate([b[h:2 * h], b[:h], b[3 * h:4 * h]])))
        ht = cell(torch.zeros(1, h), torch.tensor(hl)[None])
    np.testing.assert_allclose(out, ht[0].numpy(), atol=1e-14)


def test_treefc_equals_rnncell():
    gen = np.random.default_rng(5)
    h = 6
    p = {"W": _rand(gen, h, 2 * h), "b": _rand(gen, h)}
    hl, hr = _rand(gen, h), _rand(gen, h)
    cell = torch.nn.RNNCell(h, h, nonlinearity="tanh")
    with torch.no_grad():
        cell.weight_ih.copy_(torch.tensor(p["W"][:, h:])); cell.bias_ih.copy_(torch.tensor(p["b"]))
        cell.weight_hh.copy_(torch.tensor(p["W"][:, :h])); cell.bias_hh.zero_()
        ht = cell(torch.tensor(hr)[None], torch.tensor(hl)[None])
    np.testing.assert_allclose(cells.treefc_internal(p, hl, hr), ht[0].numpy(), atol=1e-14)


def test_lstm_chain_equals_torch_lstm():
    gen = np.random.default_rng(6)
    h, L = 4, 7
    p = {"W": _rand(gen, 4 * h, 2 * h), "b": _rand(gen, 4 * h)}
    xs = _rand(gen, L, h)
    hp, cp = np.zeros(h), np.zeros(h)
    outs = []
    for t in range(L):
        hp, cp = cells.lstm(p, xs[t], hp, cp)
        outs.append(hp)
    lstm = torch.nn.LSTM(h, h)
    with torch.no_grad():
        lstm.weight_ih_l0.copy_(torch.tensor(p["W"][:, :h])); lstm.bias_ih_l0.copy_(torch.tensor(p["b"]))
        lstm.weight_hh_l0.copy_(torch.tensor(p["W"][:, h:])); lstm.bias_hh_l0.zero_()
        yt, _ = lstm(torch.tensor(xs)[:, None, :])
    np.testing.assert_allclose(np.stack(outs), yt[:, 0].numpy(), atol=1e-13)


def test_mvrnn_identity_reduces_to_treefc():
    """A = B = I and W_M = [I/2 | I/2]: p = tanh(W [a; b] + b_W) and P = I (SURVEY pin)."""
    gen = np.random.default_rng(7)
    h = 5
    p = {"W": _rand(gen, h, 2 * h), "b": _rand(gen, h),
         "WM": np.concatenate([np.eye(h) / 2, np.eye(h) / 2], axis=1)}
    a, b = _rand(gen, h), _rand(gen, h)
    pv, P = cells.mvrnn_internal(p, a, np.eye(h), b, np.eye(h))
    np.testing.assert_allclose(pv, cells.treefc_internal(p, a, b), atol=1e-15)
    np.testing.assert_allclose(P, np.eye(h), atol=1e-15)


def test_lattice_without_words_equals_torch_lstm():
    gen = np.random.default_rng(8)
    h, L = 3, 6
    p = {"W": _rand(gen, 4 * h, 2 * h), "b": _rand(gen, 4 * h)}   # gates [i;f;o;g]
    xs = _rand(gen, L, h)
    hp, cp = np.zeros(h), np.zeros(h)
    outs = []
    for t in range(L):
        hp, cp = cells.lattice_char(p, xs[t], hp, cp, [])
        outs.append(hp)
    perm = np.concatenate([np.arange(0, h), np.arange(h, 2 * h), np.arange(3 * h, 4 * h), np.arange(2 * h, 3 * h)])
    lstm = torch.nn.LSTM(h, h)
    with torch.no_grad():
        lstm.weight_ih_l0.copy_(torch.tensor(p["W"][perm, :h])); lstm.bias_ih_l0.copy_(torch.tensor(p["b"][perm]))
        lstm.weight_hh_l0.copy_(torch.tensor(p["W"][perm, h:])); lstm.bias_hh_l0.zero_()
        yt, _ = lstm(torch.tensor(xs)[:, None, :])
    np.testing.assert_allclose(np.stack(outs), yt[:, 0].numpy(), atol=1e-13)


def test_lattice_one_word_hand_computed():
    """3 chars, one word (0 -> 2), h = 1 with hand-chosen scalars: the softmax mixing of A-23."""
    s = lambda x: 1 / (1 + np.exp(-x))
    pw = {"W": np.array([[0.5, 0.0], [0.0, 0.0], [1.0, 0.0]]), "b": np.array([0.0, 0.3, 0.0]),
          "Wl": np.array([[0.0, 2.0]]), "bl": np.array([0.1])}
    pc = {"W": np.array([[0.2, 0.0], [0.0, 0.0], [0.0, 0.0], [1.0, 0.0]]), "b": np.zeros(4)}
    hb, cb = np.array([0.0]), np.array([0.4])
    xw, xe = np.array([1.0]), np.array([0.7])
    cw, l = cells.lattice_word(pw, xw, hb, cb, xe)
    cw_hand = s(0.3) * 0.4 + s(0.5) * np.tanh(1.0)
    l_hand = s(2.0 * cw_hand + 0.1)
    np.testing.assert_allclose(cw, [cw_hand], atol=1e-15)
    np.testing.assert_allclose(l, [l_hand], atol=1e-15)
    x2 = np.array([0.9])
    hh, cc = cells.lattice_char(pc, x2, np.array([0.0]), np.array([123.0]), [(cw, l)])
    i = s(0.2 * 0.9); g = np.tanh(0.9)
    den = np.exp(i) + np.exp(l_hand)
    c_hand = np.exp(i) / den * g + np.exp(l_hand) / den * cw_hand   # c_{e-1} = 123 unused
    np.testing.assert_allclose(cc, [c_hand], atol=1e-15)
    np.testing.assert_allclose(hh, [s(0.0) * np.tanh(c_hand)], atol=1e-15)


def test_treelstm_closed_form_constant_biases():
    """All weights 0, biases constant per gate: each node carries one scalar; the recursion
    c = s(b_i)tanh(b_u) + s(b_fl)c_l + s(b_fr)c_r is evaluated here from the tree shape."""
    wl = W.treelstm(3, (2, 9), 4, "fp32", cfg=11)
    h = 4
    consts = {"L": (0.3, -0.2, 0.7), "I": (0.1, -0.4, 0.25, 0.6, -0.3)}
    for k, p in enumerate(wl.params[:2]):
        p["W"][:] = 0
        vals = consts["L" if k == 0 else "I"]
        for gi, v in enumerate(vals):
            p["b"][gi * h:(gi + 1) * h] = v
        consts["L" if k == 0 else "I"] = tuple(float(p["b"][gi * h]) for gi in range(len(vals)))
    s = lambda x: 1 / (1 + np.exp(-x))
    recs = evaluate_recursive(wl)
    for gi, g in enumerate(wl.graphs):
        memo = {}

        def cval(v):
            if v in memo:
                return memo[v]
            if g.type[v] == 0:
                bi, bo, bu = consts["L"]
                c = s(bi) * np.tanh(bu)
            else:
                l, r = g.inputs(v)
                bi, bfl, bfr, bo, bu = consts["I"]
                c = s(bi) * np.tanh(bu) + s(bfl) * cval(l) + s(bfr) * cval(r)
            memo[v] = c
            return c
        for v in range(g.num_nodes):
            if g.type[v] in (0, 1):
                bo = consts["L"][1] if g.type[v] == 0 else consts["I"][3]
                np.testing.assert_allclose(recs[gi][v]["c"], np.full(h, cval(v)), atol=1e-15)
                np.testing.assert_allclose(recs[gi][v]["h"], np.full(h, s(bo) * np.tanh(cval(v))), atol=1e-15)


def test_linear_out_selects_units():
    p = {"W": np.eye(3, 6), "b": np.array([1.0, 2.0, 3.0])}
    hv = np.arange(6.0)
    np.testing.assert_array_equal(cells.linear_out(p, hv), [1.0, 3.0, 5.0])


@pytest.mark.parametrize("wlf", [
    lambda: W.treelstm(6, (2, 12), 8, "fp32", cfg=1),
    lambda: W.treelstm(6, (2, 12), 8, "bf16", cfg=3, cell="treegru"),
    lambda: W.treefc(6, (1, 12), 8, "fp32", cfg=4),
    lambda: W.treefc(5, (1, 9), 6, "fp32", cfg=4, cell="mvrnn"),
    lambda: W.bilstm(4, (3, 9), 8, "fp32", cfg=2),
    lambda: W.lattice(5, (3, 14), 8, "fp32", cfg=5),
    lambda: W.lattice(6, (3, 14), 8, "fp32", cfg=6, cell="latticegru"),
])
def test_two_evaluators_agree(wlf):
    wl = wlf()
    a = evaluate_recursive(wl)
    b = evaluate_levels(wl)
    n = 0
    for ga, gb in zip(a, b):
        for v, ra in ga.items():
            rb = gb[v]
            for key in ("h", "c", "y", "M", "l"):
                if ra.get(key) is not None:
                    np.testing.assert_allclose(ra[key], rb[key], rtol=0, atol=1e-12)
                    n += 1
    assert n > 0



def _gru_stacked(gen, h):
    """torch GRUCell weights and the equivalent stacked [r; z; n_x; n_h] over [x; h] (A-27)."""
    wi, wh = _rand(gen, 3 * h, h), _rand(gen, 3 * h, h)
    bi, bh = _rand(gen, 3 * h), _rand(gen, 3 * h)
    W = np.zeros((4 * h, 2 * h))
    W[:h, :h], W[:h, h:] = wi[:h], wh[:h]                   # r
    W[h:2 * h, :h], W[h:2 * h, h:] = wi[h:2 * h], wh[h:2 * h]  # z
    W[2 * h:3 * h, :h] = wi[2 * h:]                          # n_x
    W[3 * h:, h:] = wh[2 * h:]                               # n_h
    b = np.concatenate([bi[:h] + bh[:h], bi[h:2 * h] + bh[h:2 * h], bi[2 * h:], bh[2 * h:]])
    cell = torch.nn.GRUCell(h, h).double()
    with torch.no_grad():
        cell.weight_ih.copy_(torch.tensor(wi)); cell.weight_hh.copy_(torch.tensor(wh))
        cell.bias_ih.copy_(torch.tensor(bi)); cell.bias_hh.copy_(torch.tensor(bh))
    return {"W": W, "b": b}, cell


def test_latticegru_word_and_wordless_char_equal_grucell():
    """A-27: the LatticeGRU word cell, and a char cell with no word ending at it, are torch GRUCell."""
    gen = np.random.default_rng(11)
    h = 6
    p, cell = _gru_stacked(gen, h)
    x, hp = _rand(gen, h), _rand(gen, h)
    with torch.no_grad():
        ref = cell(torch.tensor(x)[None], torch.tensor(hp)[None])[0].numpy()
    np.testing.assert_allclose(cells.latticegru_word(p, x, hp), ref, atol=1e-14)
    np.testing.assert_allclose(cells.latticegru_char(p, x, hp, []), ref, atol=1e-14)


def test_latticegru_char_max_pools_word_states():
    """A-27: with words ending at the char, h = element-wise max of the GRU state and the word states."""
    gen = np.random.default_rng(12)
    h = 4
    p, cell = _gru_stacked(gen, h)
    x, hp = _rand(gen, h), _rand(gen, h)
    with torch.no_grad():
        g = cell(torch.tensor(x)[None], torch.tensor(hp)[None])[0].numpy()
    w1 = np.array([10.0, -10.0, 10.0, -10.0])
    w2 = np.array([-10.0, 10.0, -10.0, -10.0])
    out = cells.latticegru_char(p, x, hp, [w1, w2])
    np.testing.assert_array_equal(out[:3], [10.0, 10.0, 10.0])
    np.testing.assert_allclose(out[3], g[3], atol=1e-14)


def test_mvrnn_cross_application_by_hand():
    """Socher et al. 2012: p = tanh(W [B a; A b] + b_W), P = W_M [A; B] -- each
    child's vector is transformed by the OTHER child's matrix, and the matrices stack A over B.
    Non-symmetric A != B and selector weights make every plausible swap visible; values by hand."""
    h = 2
    a, A = np.array([0.1, 0.2]), np.array([[1.0, 2.0], [0.0, 1.0]])
    b, B = np.array([0.3, -0.4]), np.array([[0.0, 1.0], [-1.0, 0.0]])
    I, Z = np.eye(h), np.zeros((h, h))
    # W = [I | 0] selects B a = (0.2, -0.1); W = [0 | I] selects A b = (0.3 - 0.8, -0.4) = (-0.5, -0.4)
    pv, P = cells.mvrnn_internal({"W": np.hstack([I, Z]), "b": np.zeros(h), "WM": np.hstack([I, Z])}, a, A, b, B)
    np.testing.assert_allclose(pv, np.tanh([0.2, -0.1]), rtol=0, atol=1e-15)
    np.testing.assert_allclose(P, A, rtol=0, atol=0)                       # W_M = [I | 0]: P = A
    pv, P = cells.mvrnn_internal({"W": np.hstack([Z, I]), "b": np.array([0.05, 0.0]), "WM": np.hstack([Z, I])},
                                 a, A, b, B)
    np.testing.assert_allclose(pv, np.tanh([-0.5 + 0.05, -0.4]), rtol=0, atol=1e-15)
    np.testing.assert_allclose(P, B, rtol=0, atol=0)                       # W_M = [0 | I]: P = B
    _, P = cells.mvrnn_internal({"W": np.hstack([I, I]), "b": np.zeros(h), "WM": np.hstack([I, 2 * I])}, a, A, b, B)
    np.testing.assert_allclose(P, A + 2 * B, rtol=0, atol=0)


def test_tagger_equals_torch_linear_tanh_linear():
    """BiLSTM tagger head: y = W_2 tanh(W_1 [h_f; h_b] + b_1) + b_2 is
    torch.nn.Sequential(Linear(2h, h), Tanh(), Linear(h, C)) on the concatenated states."""
    gen = np.random.default_rng(21)
    h, C = 5, 3
    p = {"W": _rand(gen, h, 2 * h), "b": _rand(gen, h), "W2": _rand(gen, C, h), "b2": _rand(gen, C)}
    hf, hb = _rand(gen, h), _rand(gen, h)
    net = torch.nn.Sequential(torch.nn.Linear(2 * h, h), torch.nn.Tanh(), torch.nn.Linear(h, C))
    with torch.no_grad():
        net[0].weight.copy_(torch.tensor(p["W"])); net[0].bias.copy_(torch.tensor(p["b"]))
        net[2].weight.copy_(torch.tensor(p["W2"])); net[2].bias.copy_(torch.tensor(p["b2"]))
        yt = net(torch.tensor(np.concatenate([hf, hb]))[None])[0].numpy()
    np.testing.assert_allclose(cells.tagger(p, hf, hb), yt, rtol=0, atol=1e-14)
    # the forward state feeds the first h columns: swapping the directions changes the logits
    assert np.max(np.abs(cells.tagger(p, hb, hf) - yt)) > 1e-3


def test_treegru_internal_mirrored_spine_equals_grucell():
    """h_l = 0, U_{.l} = 0 and b_nl = 0: internal = GRUCell(0, h_r), which pins the right-child
    path the left spine cannot see: r_r, U_nr and the h_r term of z (h_l + h_r)."""
    gen = np.random.default_rng(22)
    h = 4
    W = _rand(gen, 5 * h, 2 * h)
    W[:, :h] = 0                         # no left-child columns
    b = _rand(gen, 5 * h)
    b[3 * h:4 * h] = 0                   # a_l = U_nl h_l + b_nl = 0
    p = {"W": W, "b": b}
    hr = _rand(gen, h)
    out = cells.treegru_internal(p, np.zeros(h), hr)
    cell = torch.nn.GRUCell(h, h)
    with torch.no_grad():  # h' = (1-z) n + z h; n = tanh(r * (W_hn h + b_hn)); gates [r, z, n]
        cell.weight_ih.zero_(); cell.bias_ih.zero_()
        cell.weight_hh.copy_(torch.tensor(np.concatenate([W[2 * h:3 * h, h:], W[:h, h:], W[4 * h:, h:]])))
        cell.bias_hh.copy_(torch.tensor(np.concatenate([b[2 * h:3 * h], b[:h], b[4 * h:]])))
        ht = cell(torch.zeros(1, h), torch.tensor(hr)[None])
    np.testing.assert_allclose(out, ht[0].numpy(), rtol=0, atol=1e-14)
