"""fp64 cell equations, one node at a time — oracle, test infrastructure only.

The paper only cites the cells (Table 1); the equations below are the readings of
SURVEY Appendix A, restated in DESIGN.md §3 (A-14, A-15, A-23).  sigma = logistic.  Weights
are the logical (unpacked) parameters from workloads.make_params, upcast to fp64.
"""
from __future__ import annotations

import numpy as np


def sigmoid(x):
    return 1.0 / (1.0 + np.exp(-x))


def _f64(p, k):
    return np.asarray(p[k], dtype=np.float64)


# N-ary TreeLSTM (Tai et al.; Table 4) -------------------------------------------------

def treelstm_leaf(p, x):
    """[i;o;u] = W x + b;  c = s(i)*tanh(u);  h = s(o)*tanh(c)."""
    h = x.shape[0]
    z = _f64(p, "W") @ x + _f64(p, "b")
    i, o, u = z[:h], z[h:2 * h], z[2 * h:]
    c = sigmoid(i) * np.tanh(u)
    return sigmoid(o) * np.tanh(c), c


def treelstm_internal(p, hl, cl, hr, cr):
    """[i;f_l;f_r;o;u] = U [h_l;h_r] + b;  c = s(i)tanh(u) + s(f_l)c_l + s(f_r)c_r;  h = s(o)tanh(c)."""
    h = hl.shape[0]
    z = _f64(p, "W") @ np.concatenate([hl, hr]) + _f64(p, "b")
    i, fl, fr, o, u = (z[k * h:(k + 1) * h] for k in range(5))
    c = sigmoid(i) * np.tanh(u) + sigmoid(fl) * cl + sigmoid(fr) * cr
    return sigmoid(o) * np.tanh(c), c


def linear_out(p, h):
    """Output op O (SURVEY A-7): y = W_O h + b_O."""
    return _f64(p, "W") @ h + _f64(p, "b")


# N-ary TreeGRU (Table 4; linear-before-reset reading) ------------------

def treegru_leaf(p, x):
    """[z;n] = W x + b;  h = (1 - s(z)) * tanh(n)   (= GRUCell(x, 0) with b_hn = 0)."""
    h = x.shape[0]
    a = _f64(p, "W") @ x + _f64(p, "b")
    return (1.0 - sigmoid(a[:h])) * np.tanh(a[h:])


def treegru_internal(p, hl, hr):
    """[z;r_l;r_r] = U_g [h_l;h_r] + b_g;  a_l = U_nl h_l + b_nl;  a_r = U_nr h_r + b_nr;
    n = tanh(s(r_l)*a_l + s(r_r)*a_r);  h = (1 - s(z))*n + s(z)*(h_l + h_r).
    U_g = W[0:3h], U_nl = W[3h:4h, :h], U_nr = W[4h:5h, h:] (the other blocks are zero)."""
    h = hl.shape[0]
    W, b = _f64(p, "W"), _f64(p, "b")
    g = W[:3 * h] @ np.concatenate([hl, hr]) + b[:3 * h]
    a_l = W[3 * h:4 * h, :h] @ hl + b[3 * h:4 * h]
    a_r = W[4 * h:, h:] @ hr + b[4 * h:]
    z, rl, rr = g[:h], g[h:2 * h], g[2 * h:]
    n = np.tanh(sigmoid(rl) * a_l + sigmoid(rr) * a_r)
    return (1.0 - sigmoid(z)) * n + sigmoid(z) * (hl + hr)


# TreeFC (SURVEY A-15) and MV-RNN (Socher et al. 2012; Table 4) ----------------------------

def treefc_internal(p, hl, hr):
    """h = tanh(W [h_l;h_r] + b)."""
    return np.tanh(_f64(p, "W") @ np.concatenate([hl, hr]) + _f64(p, "b"))


def mvrnn_internal(p, a, A, bvec, B):
    """Children (a, A) and (b, B):  p = tanh(W [B a; A b] + b_W);  P = W_M [A; B]."""
    pv = np.tanh(_f64(p, "W") @ np.concatenate([B @ a, A @ bvec]) + _f64(p, "b"))
    P = _f64(p, "WM") @ np.concatenate([A, B], axis=0)
    return pv, P


# LSTM chain cells and the tagger (BiLSTM-Tagger P:286) ------------------------------------------

def lstm(p, x, hp, cp):
    """[i;f;g;o] = W [x;h_prev] + b;  c = s(f)c_prev + s(i)tanh(g);  h = s(o)tanh(c)."""
    h = x.shape[0]
    z = _f64(p, "W") @ np.concatenate([x, hp]) + _f64(p, "b")
    i, f, g, o = (z[k * h:(k + 1) * h] for k in range(4))
    c = sigmoid(f) * cp + sigmoid(i) * np.tanh(g)
    return sigmoid(o) * np.tanh(c), c


def tagger(p, hf, hb):
    """y = W_2 tanh(W_1 [h_f;h_b] + b_1) + b_2."""
    t = np.tanh(_f64(p, "W") @ np.concatenate([hf, hb]) + _f64(p, "b"))
    return _f64(p, "W2") @ t + _f64(p, "b2")


# LatticeLSTM (Zhang & Yang 2018; Fig. 7; SURVEY A-23) ------------------------------

def lattice_word(p, xw, hb, cb, xe):
    """Word cell w = (b -> e):  [i_w;f_w;g_w] = W_w [x_w;h_b] + b_w;
    c^w = s(f_w)c_b + s(i_w)tanh(g_w);  link gate l = s(W_l [x_e; c^w] + b_l).
    Returns (c^w, l)."""
    h = xw.shape[0]
    z = _f64(p, "W") @ np.concatenate([xw, hb]) + _f64(p, "b")
    i, f, g = z[:h], z[h:2 * h], z[2 * h:]
    cw = sigmoid(f) * cb + sigmoid(i) * np.tanh(g)
    l = sigmoid(_f64(p, "Wl") @ np.concatenate([xe, cw]) + _f64(p, "bl"))
    return cw, l


def lattice_char(p, x, hp, cp, words):
    """Char cell e:  [i;f;o;g] = W_c [x_e;h_{e-1}] + b_c.  No word ends at e: LSTM update
    c = s(f)c_{e-1} + s(i)tanh(g).  Otherwise c = sum_w alpha_w c^w + alpha_e tanh(g) with
    alpha = elementwise softmax over {s(i)} U {l_w}, and c_{e-1} unused (A-23).
    h = s(o)tanh(c).  ``words`` is a list of (c^w, l_w)."""
    h = x.shape[0]
    z = _f64(p, "W") @ np.concatenate([x, hp]) + _f64(p, "b")
    i, f, o, g = (z[k * h:(k + 1) * h] for k in range(4))
    if not words:
        c = sigmoid(f) * cp + sigmoid(i) * np.tanh(g)
    else:
        ei = np.exp(sigmoid(i))
        els = [np.exp(l) for _, l in words]
        den = ei + sum(els)
        c = (ei / den) * np.tanh(g)
        for (cw, _), el in zip(words, els):
            c = c + (el / den) * cw
    return sigmoid(o) * np.tanh(c), c


# LatticeGRU (A-27) ----------------------------------------------------------------

def gru(p, x, hp):
    """GRU update in torch.nn.GRUCell form with the weights stacked as one [4h, 2h] matrix over
    [x; h_prev]: rows [r; z; n_x; n_h] where the n_x rows read x only and the n_h rows h only:
    r = s(.), z = s(.), n = tanh(n_x + r * n_h), h = (1 - z) * n + z * h_prev."""
    h = x.shape[0]
    g = _f64(p, "W") @ np.concatenate([x, hp]) + _f64(p, "b")
    r, z = sigmoid(g[:h]), sigmoid(g[h:2 * h])
    n = np.tanh(g[2 * h:3 * h] + r * g[3 * h:])
    return (1.0 - z) * n + z * hp


def latticegru_word(p, xw, hb):
    """Word cell w = (b -> e): the GRU over (x_w, h_b)."""
    return gru(p, xw, hb)


def latticegru_char(p, x, hp, word_hs):
    """Char cell e: the GRU over (x_e, h_{e-1}), element-wise max-pooled with the states of the
    words ending at e (A-27)."""
    hc = gru(p, x, hp)
    for hw in word_hs:
        hc = np.maximum(hc, hw)
    return hc
