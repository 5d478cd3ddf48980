"""Encrypted HW-tiled CNN evaluation on the CPU oracle (TEST INFRASTRUCTURE ONLY).

Written from the paper, independently of ``paper_1810_00845_b200/driver.py``: it follows
Alg. 1 literally -- for every output channel, for every input channel and filter
tap: rotLeft, mulScalar, add; then one divScalar -- with only the code motion the paper
itself names ("the rotations of the input ciphertexts are invariant to the output batch and
channel, so they can be code motioned out"): each (input channel, tap) rotation is
computed once (a plain, un-hoisted rotLeft) and reused across output channels.

Lowering readings, in the order they apply:
  layout   CipherTensor metadata: C ciphertexts, valid H x W at slot
           origin + y*hS + x*wS; `clean` = every other slot is zero.
  input    the client packs the image zero-padded by the first conv's padding p (A24):
           hS = W + 2p, wS = 1, origin = p*hS + p, encoded at Delta = 2^40 at the top level.
  folding  (compile time) the 1/4 of every avgpool is folded into the next linear layer's
           weights (A26); an "act" right after a linear layer is rewritten
           a2 x^2 + a1 x + a0 = sign(a2) x'^2 + (a0 - a1^2/(4 a2)), x' = sqrt|a2| x + sqrt|a2| a1/(2 a2):
           weights * sqrt|a2|, bias beta = sqrt|a2| a1 / (2 a2) added after the linear layer's
           rescale, constant gamma = a0 - a1^2/(4 a2) added after the square's rescale (A25).
  conv     (Alg. 1) if p > 0 and the input is not clean: mask = mulPlain(x, 1 on the valid
           slots, 0 elsewhere, at scale q_top) + rescale.  Rotation amount of tap
           (i, j): origin + (i - p) hS + (j - p) wS (mod N/2).  mulScalar at pt_scale = q_top
           (A8), accumulate from the first term (A21), rescale once per output (A22),
           then add_scalar(beta).  Output layout: strides * s, origin 0, not clean (A23).
  act      rescale(mul(x, x)) (tensor + relinearize) then add_scalar(gamma), gamma
           scaled by the activation's compile-time gain (A41, see fold()).
  square   rescale(mul(x, x)).
  avgpool  x + rot(x, wS) + rot(x, hS) + rot(x, hS + wS); strides * 2 (A26).
  fc (hw input)    acc_j = sum_c mulPlain(x_c, P_jc), P_jc holding W'[j, (c, y, x)] at the valid
                   slots and 0 elsewhere (encoded at scale q_top, at x's level); rescale; then
                   rotate-and-sum acc += rot(acc, 2^t) for t < ceil(log2(span)), slot 0 holds
                   the dot product (A27, R = 1); add_scalar(beta).  Output layout "slot0".
  fc (slot0 input) out_k = sum_j mulScalar(x_j, W'[k, j]) (pt_scale q_top); rescale; add beta.
  fc, R > 1 replicas ("replicas ... in log number of rotations", A27): mask if not
                   clean; block Bk = 2^ceil(log2(span)); replicate y += rotRight(y, Bk 2^t) for
                   t < log2 R (copy r at slot offset r Bk); group g (R neurons g R + r):
                   acc_g = sum_c mulPlain(y_c, P_gc) with W'[g R + r, (c, y, x)] at slot r Bk +
                   valid slot; rescale; acc += rot(acc, 2^t) for t < log2 Bk; add beta.
                   Output layout "rep": neuron g R + r at slot r Bk of ciphertext g.
  fc (rep input)   out_k = sum_g mulPlain(z_g, Q_kg), Q_kg[r Bk] = W'[k, g R + r]; rescale;
                   acc += rot(acc, Bk 2^t) for t < log2 R; add beta.  Output "slot0".
  fire     (config 5, A33) squeeze = conv 1x1 + act; mask (the 3x3 expand's SAME padding needs
           zeros); e1 = conv 1x1 + act and e3 = conv 3x3 SAME + act on the masked
           squeeze output; output channels = e1 then e3 (concatenation is metadata).
  conv CHW (NEXT-1; layer field "chw", stride 1): mask if not clean; block stride
           CS = 2^ceil(log2(span + 2 pad_off)) with pad_off = p hS + p wS, G = (N/2) / CS channels
           per ciphertext; channel c goes to ciphertext c // G, block g = c % G, by a right
           rotation of g CS + pad_off - origin, and the channels of a ciphertext are added; per
           packed ciphertext and tap (i, j): rotLeft by (i - p) hS + (j - p) wS; per output channel:
           sum over (packed ciphertext, tap) of mulPlain with W'[oc, c, i, j] on block g's valid
           slots (scale q_top), rescale, acc += rot(acc, CS 2^t) for t < log2 G, add beta.
           Output: HW layout, origin pad_off (block 0), not clean.
  gap      global average pool: acc += rot(acc, wS 2^t) (t < log2 W), then hS 2^t (t < log2 H);
           slot 0 holds the sum; 1/(H W) folded into the preceding linear layer (A26).
"""
from __future__ import annotations

import math

import numpy as np

from .ckks import Ct, Oracle


class Layout:
    def __init__(self, kind, C, H, W, hS=0, wS=0, origin=0, clean=False, R=1, Bk=0, count=0):
        self.kind, self.C, self.H, self.W = kind, C, H, W
        self.hS, self.wS, self.origin, self.clean = hS, wS, origin, clean
        self.R, self.Bk, self.count = R, Bk, count

    def valid_slots(self):
        return [self.origin + y * self.hS + x * self.wS for y in range(self.H) for x in range(self.W)]


def fold(net: dict, weights, act_coeffs):
    """Compile-time rewrite (A25, A26, A41): per weight tensor (W', beta); per act gamma.

    A41 (compile-time gains): activation number n (execution order: "act" layers, a fire's
    squeeze then its expand) carries a gain G_n (a power of 4, default 1): the encrypted tensor
    after it holds G_n times its float64 value, so
        G_n (a2 x^2 + a1 x + a0) = x'^2 + G_n (a0 - a1^2/(4 a2)),
        x' = sqrt(a2 G_n) x + sqrt(a2 G_n) a1/(2 a2),
    and the linear layer producing x reads an input holding G_prev times its value, so its
    weights are multiplied by sqrt(a2 G_n) / G_prev.  Linear layers not followed by an act
    leave the gain unchanged; decryption divides by the output tensor's gain."""
    a0, a1, a2 = act_coeffs
    assert a2 > 0, "the folded form needs a2 > 0 (sign(a2) = +1)"
    n_acts = sum({"act": 1, "fire": 2}.get(layer[0], 0) for layer in net["layers"])
    gains = list(net.get("act_gains", [1.0] * n_acts))
    assert len(gains) == n_acts

    def act_params(n):
        G = float(gains[n])
        r = math.sqrt(a2 * G)
        return r, r * a1 / (2 * a2), G * (a0 - a1 * a1 / (4 * a2)), G

    layers = net["layers"]
    folded, gammas, wi, pools, n_act, gain = [], [], 0, 0, 0, 1.0
    _c, h, w_ = net["input"]
    for i, layer in enumerate(layers):
        nxt = layers[i + 1][0] if i + 1 < len(layers) else None
        if layer[0] == "avgpool":
            pools += 1
            h, w_ = h // 2, w_ // 2
        if layer[0] == "conv":
            _, _oc, k, st, p = layer[:5]
            h, w_ = (h + 2 * p - k) // st + 1, (w_ + 2 * p - k) // st + 1
        if layer[0] in ("conv", "fc"):
            if layer[0] == "fc":
                h, w_ = 1, 1
            wt = np.array(weights[wi], dtype=np.float64) * (0.25 ** pools)
            pools = 0
            b = 0.0
            if nxt == "act":
                r, b, gamma, G = act_params(n_act)
                n_act += 1
                wt = wt * r / gain
                gammas.append(gamma)
                gain = G
            if nxt == "gap":
                wt = wt / (h * w_)
            folded.append((wt, b))
            wi += 1
        if layer[0] == "fire":
            r1, b1, gm1, G1 = act_params(n_act)
            r2, b2, gm2, G2 = act_params(n_act + 1)
            n_act += 2
            folded.append((np.array(weights[wi], dtype=np.float64) * (0.25 ** pools) * r1 / gain, b1))
            folded.append((np.array(weights[wi + 1], dtype=np.float64) * r2 / G1, b2))
            folded.append((np.array(weights[wi + 2], dtype=np.float64) * r2 / G1, b2))
            gammas += [gm1, gm2]
            gain = G2
            pools = 0
            wi += 3
    return folded, gammas, gain


class OracleNet:
    """The network on the oracle: keys for exactly the rotation amounts the lowering uses
    (the compiler's rotation-key selection)."""

    def __init__(self, net: dict, weights, act_coeffs, seed: int = 0, nthreads=None, rot_policy: str = "exact"):
        """rot_policy "exact": one key per distinct amount; "pow2": HEAAN's default
        power-of-two keys, every rotation by k composed, least significant digit
        first, from the non-adjacent form of k -- or of k - N/2 (right rotations) when that one
        has strictly fewer non-zero digits."""
        self.net = net
        self.rot_policy = rot_policy
        self.o = Oracle(net["log_n"], net["q_bits"], net["p_bits"], seed=seed, nthreads=nthreads)
        self.folded, self.gammas, self.out_gain = fold(net, weights, act_coeffs)
        self._n_act = 0
        wanted = self._rotation_amounts()
        if rot_policy == "pow2":
            wanted = {st for k in wanted for st in self._steps(k)}
        self.amounts = sorted(wanted)
        self.o.keygen(rot_amounts=self.amounts, relin=True)

    def _steps(self, k):
        s = self.o.slots
        k %= s
        if k == 0:
            return []

        def naf_digits(v):                       # signed-binary digits, least significant first
            digits = []
            pos = 0
            while v != 0:
                if v % 2 == 0:
                    d = 0
                else:
                    d = 2 - (v % 4)              # v = 1 mod 4 -> +1, v = 3 mod 4 -> -1
                    v -= d
                if d:
                    digits.append(d * 2 ** pos)
                v //= 2
                pos += 1
            return digits
        a, b = naf_digits(k), naf_digits(k - s)
        return [d % s for d in (b if len(b) < len(a) else a)]

    def _rot(self, ct, k):
        """rotLeft under the key policy: one key switch (exact) or the composition (pow2)."""
        o = self.o
        if self.rot_policy == "exact":
            return o.rot_left(ct, k)
        steps = self._steps(k)
        if not steps:
            return o.copy(ct)
        for st in steps:
            ct = o.rot_left(ct, st)
        return ct

    # ---- layout walk (same walk as forward, metadata only) -------------------------------
    def _input_layout(self):
        c, h, w = self.net["input"]
        first = self.net["layers"][0]
        p = first[4] if first[0] == "conv" else 0
        hs = w + 2 * p
        return Layout("hw", c, h, w, hS=hs, wS=1, origin=p * hs + p, clean=True)

    def _rotation_amounts(self):
        s = self.o.slots
        lay = self._input_layout()
        amts = set()
        for layer in self.net["layers"]:
            kind = layer[0]
            if kind == "conv" and len(layer) > 5 and layer[5] == "chw":
                _, oc, k, st, p = layer[:5]
                pad_off = p * lay.hS + p * lay.wS
                span = (lay.H - 1) * lay.hS + (lay.W - 1) * lay.wS + 1
                cs = 2 ** math.ceil(math.log2(span + 2 * pad_off))
                G = max(1, s // cs)
                for g in range(min(G, lay.C)):
                    amts.add((s - (g * cs + pad_off - lay.origin) % s) % s)
                for i in range(k):
                    for j in range(k):
                        amts.add(((i - p) * lay.hS + (j - p) * lay.wS) % s)
                amts.update(cs * 2 ** t for t in range(int(math.log2(G))))
                lay = Layout("hw", oc, lay.H, lay.W, lay.hS, lay.wS, pad_off, False)
            elif kind == "conv":
                _, oc, k, st, p = layer[:5]
                for i in range(k):
                    for j in range(k):
                        amts.add((lay.origin + (i - p) * lay.hS + (j - p) * lay.wS) % s)
                lay = Layout("hw", oc, (lay.H + 2 * p - k) // st + 1, (lay.W + 2 * p - k) // st + 1,
                             lay.hS * st, lay.wS * st, 0, False)
            elif kind == "avgpool":
                amts.update({lay.wS % s, lay.hS % s, (lay.hS + lay.wS) % s})
                lay = Layout("hw", lay.C, lay.H // 2, lay.W // 2, lay.hS * 2, lay.wS * 2, lay.origin, False)
            elif kind == "fire":
                for i in range(3):
                    for j in range(3):
                        amts.add((lay.origin + (i - 1) * lay.hS + (j - 1) * lay.wS) % s)
                amts.add(lay.origin % s)
                lay = Layout("hw", layer[2] + layer[3], lay.H, lay.W, lay.hS, lay.wS, lay.origin, False)
            elif kind == "gap":
                amts.update(lay.wS * 2 ** t for t in range(int(math.log2(lay.W))))
                amts.update(lay.hS * 2 ** t for t in range(int(math.log2(lay.H))))
                lay = Layout("slot0", lay.C, 1, 1)
            elif kind == "fc" and lay.kind == "hw" and len(layer) > 3 and layer[3] == "chw":
                span = (lay.H - 1) * lay.hS + (lay.W - 1) * lay.wS + 1
                cs = 2 ** math.ceil(math.log2(span))
                G = min(max(1, s // cs), 2 ** math.ceil(math.log2(max(1, lay.C))))
                for g in range(min(G, lay.C)):
                    amts.add((s - (g * cs - lay.origin) % s) % s)
                amts.update(2 ** t for t in range(int(math.log2(G * cs))))
                lay = Layout("slot0", layer[1], 1, 1)
            elif kind == "fc" and lay.kind == "hw" and len(layer) > 2 and layer[2] > 1:
                R = layer[2]
                span = lay.origin + (lay.H - 1) * lay.hS + (lay.W - 1) * lay.wS + 1
                bk = 2 ** math.ceil(math.log2(span))
                amts.update((s - bk * 2 ** t) % s for t in range(int(math.log2(R))))
                amts.update(2 ** t for t in range(int(math.log2(bk))))
                lay = Layout("rep", -(-layer[1] // R), 1, 1, R=R, Bk=bk, count=layer[1])
            elif kind == "fc" and lay.kind == "rep":
                amts.update(lay.Bk * 2 ** t for t in range(int(math.log2(lay.R))))
                lay = Layout("slot0", layer[1], 1, 1)
            elif kind == "fc" and lay.kind == "hw":
                span = lay.origin + (lay.H - 1) * lay.hS + (lay.W - 1) * lay.wS + 1
                amts.update(1 << t for t in range(math.ceil(math.log2(span))))
                lay = Layout("slot0", layer[1], 1, 1)
            elif kind == "fc":
                lay = Layout("slot0", layer[1], 1, 1)
        amts.discard(0)
        return amts

    # ---- client ---------------------------------------------------------------------------
    def encrypt_image(self, image: np.ndarray):
        lay = self._input_layout()
        cts = []
        for c in range(lay.C):
            v = np.zeros(self.o.slots)
            for y in range(lay.H):
                for x in range(lay.W):
                    v[lay.origin + y * lay.hS + x * lay.wS] = image[c, y, x]
            cts.append(self.o.encrypt(self.o.encode(v, self.net["scale"])))
        return cts, lay

    def decrypt_output(self, cts, lay) -> np.ndarray:
        """Decrypt + decode the network output, divided by its compile-time gain (A41)."""
        vals = [self.o.decode(self.o.decrypt(ct)) / self.out_gain for ct in cts]
        if lay.kind == "slot0":
            return np.array([v[0] for v in vals])
        if lay.kind == "rep":
            flat = [v[r * lay.Bk] for v in vals for r in range(lay.R)]
            return np.array(flat[:lay.count])
        sl = lay.valid_slots()
        return np.array([[v[i] for i in sl] for v in vals]).reshape(lay.C, lay.H, lay.W)

    # ---- server ---------------------------------------------------------------------------
    def _mask(self, cts, lay):
        o = self.o
        m = np.zeros(o.slots)
        m[lay.valid_slots()] = 1.0
        out = []
        for ct in cts:
            pt = o.encode(m, float(o.q[ct.level]), ct.level)
            out.append(o.rescale(o.mul_plain(ct, pt)))
        lay = Layout(lay.kind, lay.C, lay.H, lay.W, lay.hS, lay.wS, lay.origin, True)
        return out, lay

    def conv(self, cts, lay, layer, w, beta):
        """Alg. 1 with the rotations code-motioned out of the oc loop."""
        if len(layer) > 5 and layer[5] == "chw":
            return self.conv_chw(cts, lay, layer, w, beta)
        o = self.o
        _, oc_n, k, st, p = layer[:5]
        if p > 0 and not lay.clean:
            cts, lay = self._mask(cts, lay)
        rotated = {}
        for ic in range(lay.C):
            for i in range(k):
                for j in range(k):
                    rotated[ic, i, j] = self._rot(cts[ic], lay.origin + (i - p) * lay.hS + (j - p) * lay.wS)
        outs = []
        for oc in range(oc_n):
            acc = None                                   # zeroCipher (A21)
            for ic in range(lay.C):
                for i in range(k):
                    for j in range(k):
                        temp = o.mul_scalar(rotated[ic, i, j], float(w[oc, ic, i, j]))
                        acc = temp if acc is None else o.add(acc, temp)
            acc = o.div_scalar(acc, o.max_scalar_div(acc, 1 << 62))
            if beta:
                acc = o.add_scalar(acc, beta)
            outs.append(acc)
        nl = Layout("hw", oc_n, (lay.H + 2 * p - k) // st + 1, (lay.W + 2 * p - k) // st + 1,
                    lay.hS * st, lay.wS * st, 0, False)
        return outs, nl

    def conv_chw(self, cts, lay, layer, w, beta):
        o = self.o
        _, oc_n, k, st, p = layer[:5]
        assert st == 1, "CHW conv: stride 1"
        if not lay.clean:
            cts, lay = self._mask(cts, lay)
        s = o.slots
        pad_off = p * lay.hS + p * lay.wS
        span = (lay.H - 1) * lay.hS + (lay.W - 1) * lay.wS + 1
        cs = 2 ** math.ceil(math.log2(span + 2 * pad_off))
        G = max(1, s // cs)
        C = lay.C
        npk = -(-C // G)
        packed = []
        for kk in range(npk):
            acc = None
            for g in range(G):
                c = kk * G + g
                if c >= C:
                    break
                shift = (g * cs + pad_off - lay.origin) % s
                r = self._rot(cts[c], (s - shift) % s)
                acc = r if acc is None else o.add(acc, r)
            packed.append(acc)
        rel = [y * lay.hS + x * lay.wS for y in range(lay.H) for x in range(lay.W)]
        rot = {}
        for kk in range(npk):
            for i in range(k):
                for j in range(k):
                    rot[kk, i, j] = self._rot(packed[kk], (i - p) * lay.hS + (j - p) * lay.wS)
        outs = []
        for oc in range(oc_n):
            acc = None
            for kk in range(npk):
                for i in range(k):
                    for j in range(k):
                        v = np.zeros(s)
                        for g in range(G):
                            c = kk * G + g
                            if c < C:
                                for r_ in rel:
                                    v[g * cs + pad_off + r_] = w[oc, c, i, j]
                        x = rot[kk, i, j]
                        term = o.mul_plain(x, o.encode(v, float(o.q[x.level]), x.level))
                        acc = term if acc is None else o.add(acc, term)
            acc = o.rescale(acc)
            for t in range(int(math.log2(G))):
                acc = o.add(acc, self._rot(acc, cs * 2 ** t))
            if beta:
                acc = o.add_scalar(acc, beta)
            outs.append(acc)
        return outs, Layout("hw", oc_n, lay.H, lay.W, lay.hS, lay.wS, pad_off, False)

    def act(self, cts, lay, square_only=False):
        o = self.o
        out = []
        gamma = 0.0
        if not square_only:
            gamma = self.gammas[self._n_act]
            self._n_act += 1
        for ct in cts:
            y = o.rescale(o.mul(ct, ct))
            if gamma:
                y = o.add_scalar(y, gamma)
            out.append(y)
        return out, Layout(lay.kind, lay.C, lay.H, lay.W, lay.hS, lay.wS, lay.origin, False, lay.R, lay.Bk,
                           lay.count)

    def avgpool(self, cts, lay):
        o = self.o
        out = []
        for ct in cts:
            y = o.add(ct, self._rot(ct, lay.wS))
            y = o.add(y, self._rot(ct, lay.hS))
            y = o.add(y, self._rot(ct, lay.hS + lay.wS))
            out.append(y)
        return out, Layout("hw", lay.C, lay.H // 2, lay.W // 2, lay.hS * 2, lay.wS * 2, lay.origin, False)

    def fc_replicas(self, cts, lay, layer, w, beta):
        o = self.o
        n_out, R = layer[1], layer[2]
        if not lay.clean:
            cts, lay = self._mask(cts, lay)
        span = lay.origin + (lay.H - 1) * lay.hS + (lay.W - 1) * lay.wS + 1
        bk = 2 ** math.ceil(math.log2(span))
        assert R * bk <= o.slots
        ys = []
        for ct in cts:
            y = ct
            for t in range(int(math.log2(R))):
                y = o.add(y, self._rot(y, o.slots - bk * 2 ** t))      # right rotation
            ys.append(y)
        sl = lay.valid_slots()
        hw = lay.H * lay.W
        groups = -(-n_out // R)
        outs = []
        for g in range(groups):
            acc = None
            for c in range(lay.C):
                v = np.zeros(o.slots)
                for r in range(R):
                    if g * R + r < n_out:
                        for i, slot in enumerate(sl):
                            v[r * bk + slot] = w[g * R + r, c * hw + i]
                pt = o.encode(v, float(o.q[ys[c].level]), ys[c].level)
                term = o.mul_plain(ys[c], pt)
                acc = term if acc is None else o.add(acc, term)
            acc = o.rescale(acc)
            for t in range(int(math.log2(bk))):
                acc = o.add(acc, self._rot(acc, 2 ** t))
            if beta:
                acc = o.add_scalar(acc, beta)
            outs.append(acc)
        return outs, Layout("rep", groups, 1, 1, R=R, Bk=bk, count=n_out)

    def fc_chw(self, cts, lay, layer, w, beta):
        """CHW-tiled matmul (NEXT-1): mask, move channel c to block c mod G of
        packed ciphertext c div G (blocks of cs slots, cs = span rounded up to a power of two),
        then per neuron: sum over packed ciphertexts of mulPlain with the neuron's weights on every
        block, rescale, rotate-and-sum by 1, 2, 4, ... < G cs into slot 0."""
        o = self.o
        n_out = layer[1]
        if not lay.clean:
            cts, lay = self._mask(cts, lay)
        s = o.slots
        span = (lay.H - 1) * lay.hS + (lay.W - 1) * lay.wS + 1
        cs = 2 ** math.ceil(math.log2(span))
        G = min(max(1, s // cs), 2 ** math.ceil(math.log2(max(1, lay.C))))
        C = lay.C
        packed = []
        for kk in range(-(-C // G)):
            acc = None
            for g in range(G):
                c = kk * G + g
                if c >= C:
                    break
                r = self._rot(cts[c], (s - (g * cs - lay.origin) % s) % s)
                acc = r if acc is None else o.add(acc, r)
            packed.append(acc)
        rel = [y * lay.hS + x * lay.wS for y in range(lay.H) for x in range(lay.W)]
        hw = lay.H * lay.W
        outs = []
        for jo in range(n_out):
            acc = None
            for kk, x in enumerate(packed):
                v = np.zeros(s)
                for g in range(G):
                    c = kk * G + g
                    if c < C:
                        for i, r_ in enumerate(rel):
                            v[g * cs + r_] = w[jo, c * hw + i]
                term = o.mul_plain(x, o.encode(v, float(o.q[x.level]), x.level))
                acc = term if acc is None else o.add(acc, term)
            acc = o.rescale(acc)
            for t in range(int(math.log2(G * cs))):
                acc = o.add(acc, self._rot(acc, 2 ** t))
            if beta:
                acc = o.add_scalar(acc, beta)
            outs.append(acc)
        return outs, Layout("slot0", n_out, 1, 1)

    def fc(self, cts, lay, layer, w, beta):
        o = self.o
        n_out = layer[1]
        outs = []
        if lay.kind == "hw" and len(layer) > 3 and layer[3] == "chw":
            return self.fc_chw(cts, lay, layer, w, beta)
        if lay.kind == "hw" and len(layer) > 2 and layer[2] > 1:
            return self.fc_replicas(cts, lay, layer, w, beta)
        if lay.kind == "rep":
            for k in range(n_out):
                acc = None
                for g, ct in enumerate(cts):
                    v = np.zeros(o.slots)
                    for r in range(lay.R):
                        if g * lay.R + r < lay.count:
                            v[r * lay.Bk] = w[k, g * lay.R + r]
                    term = o.mul_plain(ct, o.encode(v, float(o.q[ct.level]), ct.level))
                    acc = term if acc is None else o.add(acc, term)
                acc = o.rescale(acc)
                for t in range(int(math.log2(lay.R))):
                    acc = o.add(acc, self._rot(acc, lay.Bk * 2 ** t))
                if beta:
                    acc = o.add_scalar(acc, beta)
                outs.append(acc)
            return outs, Layout("slot0", n_out, 1, 1)
        if lay.kind == "hw":
            sl = lay.valid_slots()
            span = lay.origin + (lay.H - 1) * lay.hS + (lay.W - 1) * lay.wS + 1
            steps = math.ceil(math.log2(span))
            hw = lay.H * lay.W
            for jo in range(n_out):
                acc = None
                for c in range(lay.C):
                    v = np.zeros(o.slots)
                    v[sl] = w[jo, c * hw:(c + 1) * hw]
                    pt = o.encode(v, float(o.q[cts[c].level]), cts[c].level)
                    term = o.mul_plain(cts[c], pt)
                    acc = term if acc is None else o.add(acc, term)
                acc = o.rescale(acc)
                for t in range(steps):
                    acc = o.add(acc, self._rot(acc, 1 << t))
                if beta:
                    acc = o.add_scalar(acc, beta)
                outs.append(acc)
        else:
            for ko in range(n_out):
                acc = None
                for jn, ct in enumerate(cts):
                    term = o.mul_scalar(ct, float(w[ko, jn]))
                    acc = term if acc is None else o.add(acc, term)
                acc = o.rescale(acc)
                if beta:
                    acc = o.add_scalar(acc, beta)
                outs.append(acc)
        return outs, Layout("slot0", n_out, 1, 1)

    def fire(self, cts, lay, layer, f3):
        _, sq, e1, e3 = layer
        (wsq, bsq), (we1, b1), (we3, b3) = f3
        s, ls = self.conv(cts, lay, ("conv", sq, 1, 1, 0), wsq, bsq)
        s, ls = self.act(s, ls)
        s, ls = self._mask(s, ls)
        x1, l1 = self.conv(s, ls, ("conv", e1, 1, 1, 0), we1, b1)
        x3, _l3 = self.conv(s, ls, ("conv", e3, 3, 1, 1), we3, b3)
        out, lo = self.act(x1 + x3, l1)          # one activation (one gain, A41) on the concatenation
        return out, Layout("hw", e1 + e3, lo.H, lo.W, lo.hS, lo.wS, lo.origin, False)

    def gap(self, cts, lay):
        o = self.o
        out = []
        for ct in cts:
            acc = ct
            for t in range(int(math.log2(lay.W))):
                acc = o.add(acc, self._rot(acc, lay.wS * 2 ** t))
            for t in range(int(math.log2(lay.H))):
                acc = o.add(acc, self._rot(acc, lay.hS * 2 ** t))
            out.append(acc)
        return out, Layout("slot0", lay.C, 1, 1)

    def forward(self, cts, lay, trace=None, stop_after=None):
        """Server-side evaluation; `trace` (a list) receives (layer index, ciphertexts) after
        every layer for per-layer parity checks; `stop_after` = last layer index to evaluate
        (sampled parity of networks too large for the oracle end to end)."""
        wi = 0
        self._n_act = 0
        for li, layer in enumerate(self.net["layers"]):
            if stop_after is not None and li > stop_after:
                break
            kind = layer[0]
            if kind == "conv":
                w, b = self.folded[wi]
                wi += 1
                cts, lay = self.conv(cts, lay, layer, w, b)
            elif kind == "fc":
                w, b = self.folded[wi]
                wi += 1
                cts, lay = self.fc(cts, lay, layer, w, b)
            elif kind == "act":
                cts, lay = self.act(cts, lay)
            elif kind == "square":
                cts, lay = self.act(cts, lay, square_only=True)
            elif kind == "avgpool":
                cts, lay = self.avgpool(cts, lay)
            elif kind == "fire":
                cts, lay = self.fire(cts, lay, layer, self.folded[wi:wi + 3])
                wi += 3
            elif kind == "gap":
                cts, lay = self.gap(cts, lay)
            else:
                raise ValueError(kind)
            if trace is not None:
                trace.append((li, list(cts)))
        return cts, lay
