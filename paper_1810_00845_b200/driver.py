"""HW-tiled encrypted CNN driver on libhisa.

The CHET runtime's homomorphic tensor kernels lowered onto the HISA calls of
``hisa.py`` -- argument marshalling and layout bookkeeping only; every ciphertext word is
produced by the sm_100a kernels behind the C-ABI.

  * CipherTensor metadata: C ciphertexts (HW-tiling), valid H x W at slot
    origin + y*hS + x*wS, `clean` = zeros outside the valid slots.
  * conv2d = Alg. 1: the IC*K^2 rotations are hoisted out of the output-channel
    loop AND share one ModUp per input channel (hisa_rot_left_hoisted, K7); the
    mulScalar + add accumulation over all (ic, tap) for all OC outputs is ONE fused kernel
    (hisa_conv_accumulate, K8); one divScalar per output.
  * activation a0 + a1 x + a2 x^2 (A25) folded to sign(a2) x'^2 + const: one level;
    per-activation compile-time gains (A41) keep small signals above the CKKS noise floor.
  * 2x2 average pool: three hoisted rotations + adds, 1/4 folded forward (A26).
  * FC / matmul (A27, R = 1): mulPlain per input channel, rescale, rotate-and-sum
    with every output neuron's rotation batched under one key (hisa_rot_left_batch).
  * multi-GPU: input channels of every conv / FC are partitioned across ranks;
    each rank accumulates partial sums for ALL outputs (hisa_conv_accumulate_dev into a torch
    int64 buffer), one NCCL reduce-scatter (int64 SUM, exact: partials < 2^60, <= 8 ranks)
    hands every rank its own output channels, hisa_ct_adopt_sum reduces them mod q_i, and the
    owner rescales / activates -- its outputs are exactly its input shard of the next layer.

The lowering is written down in DESIGN.md section 5 and implemented independently (without
shared code) by oracle/nets.py; ciphertexts are compared bit for bit by tests/test_driver.py.

A symbolic backend (`Symbolic`) executes the same driver on metadata only -- the paper's
symbolic analysers: it yields the level plan, the distinct rotation amounts for
key generation and the operation counts, and never touches ciphertext data.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, replace

import numpy as np


# ------------------------------------------------------------------------------ layouts
@dataclass(frozen=True)
class Layout:
    """CipherTensor metadata.  kind "hw": channel c's valid H x W plane at slots
    origin + y*hS + x*wS; kind "slot0": one value per ciphertext, in slot 0."""
    kind: str
    C: int
    H: int = 1
    W: int = 1
    hS: int = 0
    wS: int = 0
    origin: int = 0
    clean: bool = False
    count: int = 0       # kind "rep": number of valid values (R per ciphertext at slots r * hS)

    def slots_of_valid(self) -> np.ndarray:
        y, x = np.meshgrid(np.arange(self.H), np.arange(self.W), indexing="ij")
        return (self.origin + y * self.hS + x * self.wS).ravel()

    def span(self) -> int:
        return self.origin + (self.H - 1) * self.hS + (self.W - 1) * self.wS + 1


def act_fold(coeffs, gain: float = 1.0):
    """A25 with a compile-time output gain G (A41): G (a2 x^2 + a1 x + a0) = x'^2 + gamma with
    x' = r x + beta, r = sqrt(a2 G), beta = r a1 / (2 a2), gamma = G (a0 - a1^2 / (4 a2))
    (a2 > 0).  G = 1 is the plain fold."""
    a0, a1, a2 = coeffs
    if not a2 > 0:
        raise ValueError("folded activation needs a2 > 0")
    r = math.sqrt(a2 * gain)
    return r, r * a1 / (2 * a2), gain * (a0 - a1 * a1 / (4 * a2))


def act_gains(net: dict):
    """A41: the compile-time gain of every activation in execution order ("act" layers; a fire
    module's squeeze then its expand), powers of 4 (so sqrt(a2 G) = sqrt(a2) 2^e and every
    weight rewrite below is exact in any order); default 1."""
    n_act = sum(1 if layer[0] == "act" else 2 if layer[0] == "fire" else 0 for layer in net["layers"])
    gains = [float(g) for g in net.get("act_gains", [1.0] * n_act)]
    if len(gains) != n_act:
        raise ValueError(f"act_gains: {len(gains)} given, the net has {n_act} activations")
    for g in gains:
        m, e = math.frexp(g)
        if m != 0.5 or (e - 1) % 2:
            raise ValueError(f"act gain {g} is not a power of 4")
    return gains


def compile_weights(net: dict, weights, act_coeffs):
    """Compile-time weight rewriting: avg-pool 1/4 factors pushed into the next linear layer
    (A26), the global-average-pool 1/(H W) into the linear layer before it (A26), and the
    activation scale / bias folded into the preceding linear layer (A25; a fire module's three
    convs are each followed by an activation).  With activation gains (A41) every encrypted
    tensor holds G x its float64 value: a linear layer followed by an activation of gain G_out
    divides its weights by the gain G_in of its input and folds r = sqrt(a2 G_out); any other
    linear layer keeps the gain.
    Returns ([(W', beta)] per weight tensor, in order, [gamma] per activation, [(gain, offset)]
    per layer: the layer's encrypted output holds gain x value + offset (a linear layer feeding
    an activation holds its folded x' = r x + beta))."""
    gains = iter(act_gains(net))
    layers = net["layers"]
    out, gammas, layer_affine, pending, it, g_cur = [], [], [], 1.0, iter(weights), 1.0
    c, h, w = net["input"]
    for i, layer in enumerate(layers):
        kind = layer[0]
        if kind == "avgpool":
            pending *= 0.25
            h, w = h // 2, w // 2
        elif kind in ("conv", "fc"):
            nxt = layers[i + 1][0] if i + 1 < len(layers) else None
            if kind == "conv":
                _, oc, k, st, p = layer[:5]
                h, w = (h + 2 * p - k) // st + 1, (w + 2 * p - k) // st + 1
                c = oc
            else:
                c, h, w = layer[1], 1, 1
            if nxt == "act":
                g_out = next(gains)
                r, beta, gamma = act_fold(act_coeffs, g_out)
                gammas.append(gamma)
                f = pending * r / g_cur
                g_cur = g_out
                affine = (r, beta)
            else:
                f, beta = pending, 0.0
                affine = (g_cur, 0.0)
            if nxt == "gap":
                f = f * (1.0 / (h * w))
                affine = (affine[0] / (h * w), 0.0)       # the gap's 1/(H W) folded in (A26)
            out.append((np.asarray(next(it), dtype=np.float64) * f, beta))
            pending = 1.0
        elif kind == "fire":
            g_sq, g_ex = next(gains), next(gains)
            r_sq, beta_sq, gamma_sq = act_fold(act_coeffs, g_sq)
            r_ex, beta_ex, gamma_ex = act_fold(act_coeffs, g_ex)
            out.append((np.asarray(next(it), dtype=np.float64) * (pending * r_sq / g_cur), beta_sq))  # squeeze
            out.append((np.asarray(next(it), dtype=np.float64) * (r_ex / g_sq), beta_ex))             # expand 1x1
            out.append((np.asarray(next(it), dtype=np.float64) * (r_ex / g_sq), beta_ex))             # expand 3x3
            gammas += [gamma_sq, gamma_ex]
            pending, g_cur = 1.0, g_ex
            c = layer[2] + layer[3]
        # a pool's 1/4 is folded forward (A26): its output holds the sum, g_cur / pending x the mean
        layer_affine.append(affine if kind in ("conv", "fc") else (g_cur / pending, 0.0))
    return out, gammas, layer_affine


def input_layout(net: dict) -> Layout:
    """The client's packing (A24): zero padding of the first conv materialised."""
    c, h, w = net["input"]
    first = net["layers"][0]
    p = first[4] if first[0] == "conv" else 0
    hs = w + 2 * p
    return Layout("hw", c, h, w, hs, 1, p * hs + p, True)


# ------------------------------------------------------------------------------ symbolic backend
class Symbolic:
    """Metadata-only HISA backend (the paper's symbolic analysers)."""

    def __init__(self, log_n: int, moduli):
        self.slots = (1 << log_n) // 2
        self.q = list(moduli)
        self.cts = {}
        self.next = 1
        self.rotations = set()
        self.rot_level = {}       # amount -> highest level it is used at (key truncation)
        self.counts = {}

    def _new(self, level, scale):
        h = self.next
        self.next += 1
        self.cts[h] = (level, scale)
        return h

    def _rot(self, kk, lv):
        self.rotations.add(kk)          # (lv = -1: an empty batch on a rank without channels)
        self.rot_level[kk] = max(lv, self.rot_level.get(kk, -1))

    def _count(self, op, n=1):
        self.counts[op] = self.counts.get(op, 0) + n

    def ct_info(self, h):
        lv, sc = self.cts[h]
        return lv, 2, sc

    def free(self, h):
        self.cts.pop(h, None)

    def fresh(self, level, scale):
        return self._new(level, scale)

    def rot_left_hoisted(self, h, ks):
        lv, sc = self.cts[h]
        out = []
        for k in ks:
            kk = k % self.slots
            if kk:
                self._rot(kk, lv)
                self._count("rot_hoisted")
            out.append(self._new(lv, sc))
        return out

    def rot_left_hoisted_batch(self, hs, ks):
        return [self.rot_left_hoisted(h, ks) for h in hs]

    def rot_left_batch(self, hs, k):
        kk = k % self.slots
        if kk:
            self._rot(kk, max((self.cts[h][0] for h in hs), default=-1))
            self._count("rot", len(hs))
        return [self._new(*self.cts[h]) for h in hs]

    def conv_accumulate(self, hs, W, pt_scale=0.0):
        lv, sc = self.cts[hs[0]]
        n_out = len(W) // len(hs)
        self._count("scalar_mac_ct", len(W))
        return [self._new(lv, sc * float(self.q[lv])) for _ in range(n_out)]

    def rescale(self, h):
        lv, sc = self.cts[h]
        if lv == 0:
            raise RuntimeError("level budget exhausted (MODULUS_EXHAUSTED)")
        self._count("rescale")
        return self._new(lv - 1, sc / float(self.q[lv]))

    def mul(self, a, b):
        lv, sa = self.cts[a]
        self._count("mul_relin")
        return self._new(lv, sa * self.cts[b][1])

    def add(self, a, b):
        self._count("add")
        return self._new(*self.cts[a])

    def add_scalar(self, a, x):
        return self._new(*self.cts[a])

    def copy(self, a):
        return self._new(*self.cts[a])

    def mul_batch(self, a, b):
        return [self.mul(x, y) for x, y in zip(a, b)]

    def rescale_batch(self, hs):
        return [self.rescale(h) for h in hs]

    def rot_add_batch(self, hs, k):
        kk = k % self.slots
        if kk:
            self._rot(kk, max((self.cts[h][0] for h in hs), default=-1))
            self._count("rot", len(hs))
        self._count("add", len(hs))
        return [self._new(*self.cts[h]) for h in hs]

    def mul_plain_accumulate(self, hs, pts, J):
        lv, sc = self.cts[hs[0]]
        self._count("mul_plain", len(pts))
        return [self._new(lv, sc * pts[0][2]) for _ in range(J)]

    def encode(self, v, scale, level):
        self._count("encode")
        return ("pt", level, scale)

    def encode_batch(self, vs, scale, level):
        return [self.encode(v, scale, level) for v in vs]

    def mul_plain(self, a, p):
        lv, sc = self.cts[a]
        self._count("mul_plain")
        return self._new(lv, sc * p[2])


# ------------------------------------------------------------------------------ the network
class EncryptedNet:
    """One network on one backend (a hisa.Context, or Symbolic for planning).

    `group` (torch.distributed process group, optional) shards every linear layer's input
    channels across ranks; None = single GPU."""

    def __init__(self, backend, net: dict, weights, act_coeffs, group=None, rot_policy: str = "exact",
                 partition: str = "ic", exchange_at_world1: bool = False):
        """rot_policy: "exact" = one key per distinct rotation amount, chosen by the compiler
        (CHET); "pow2" = HEAAN's default power-of-two keys (left and right),
        every other amount composed from them (the baseline of the paper's Fig. rotopt).
        partition (multi-GPU convs): "ic" = input channels sharded, partial sums for
        all outputs reduce-scattered (each hoisted rotation computed once); "oc" = the north
        star's output-channel partition: the layer's inputs all-gathered, every rank rotates all
        of them and accumulates its own output channels (the measured baseline).  FC layers
        always follow 8e's plan: inputs all-gathered, output neurons / R-groups partitioned."""
        if rot_policy not in ("exact", "pow2"):
            raise ValueError(rot_policy)
        if partition not in ("ic", "oc"):
            raise ValueError(partition)
        self.partition = partition
        self.rot_policy = rot_policy
        self.b = backend
        self.net = net
        self.folded, self.gammas, self.layer_affine = compile_weights(net, weights, act_coeffs)
        self._act_i = 0
        self.slots = backend.slots
        self.q = list(backend.q)
        self._pts = {}
        self.group = group
        if group is not None:
            import torch.distributed as dist
            self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        else:
            self.rank, self.world = 0, 1
        # the exchange code path (reduce-scatter / all-gather, adoption of the int64 sums) runs
        # when there is more than one rank -- or, on request, on a one-rank group: the only way
        # to drive the NCCL data plane on a single-GPU box (tests/test_nccl_world1.py)
        self.sharded = self.world > 1 or (group is not None and exchange_at_world1)

    # ---- planning (symbolic execution) ------------------------------------------------------
    @staticmethod
    def plan(net: dict, weights, act_coeffs, moduli, rot_policy: str = "exact"):
        """Level plan, distinct rotation amounts (keygen input), op counts."""
        sym = Symbolic(net["log_n"], moduli)
        en = EncryptedNet(sym, net, weights, act_coeffs, rot_policy=rot_policy)
        lay = input_layout(net)
        top = len(moduli) - 2
        cts = [sym.fresh(top, net["scale"]) for _ in range(lay.C)]
        outs, out_lay = en.forward(cts, lay)
        final = sym.cts[outs[0]][0]
        return {"rotations": sorted(sym.rotations), "rotation_levels": dict(sorted(sym.rot_level.items())),
                "final_level": final, "levels_used": top - final, "counts": dict(sym.counts), "out_layout": out_lay}

    @staticmethod
    def keygen(backend, plan, relin: bool = True):
        """Keys for a plan: the relinearisation key and one rotation key per amount, each rotation
        key truncated to the highest level the network rotates by it (hisa_keygen max_level;
        SURVEY 7 hard part 3 -- 600 MiB per full key at N = 2^16, L = 24)."""
        by_level = {}
        for k, lv in plan["rotation_levels"].items():
            by_level.setdefault(lv, []).append(k)
        backend.keygen([], relin)
        for lv, ks in sorted(by_level.items()):
            backend.keygen(ks, False, lv)

    # ---- sharding ---------------------------------------------------------------
    def owned(self, n: int) -> range:
        """Contiguous block of channel indices owned by this rank (rank r gets block r)."""
        per = -(-n // self.world)
        return range(min(n, self.rank * per), min(n, (self.rank + 1) * per))

    # ---- client ---------------------------------------------------------------------------
    def encrypt_image(self, image):
        """Encode + encrypt the packed image (client side), one ciphertext per channel."""
        lay = input_layout(self.net)
        cts = []
        for c in range(lay.C):
            v = np.zeros(self.slots)
            v[lay.slots_of_valid()] = np.asarray(image[c], dtype=np.float64).ravel()
            pt = self.b.encode(v, self.net["scale"], -1)
            cts.append(self.b.encrypt(pt))
            self.b.free(pt)
        return cts, lay

    def decrypt_output(self, cts, lay, affine=None) -> np.ndarray:
        """Decrypt + decode, undoing the tensor's compile-time (gain, offset) (A41; default: the
        network output's; an intermediate layer li passes self.layer_affine[li])."""
        g, off = self.layer_affine[-1] if affine is None else affine
        pts = [self.b.decrypt(ct) for ct in cts]
        if hasattr(self.b, "decode_batch"):      # GPU decode of all outputs at once (NEXT-4)
            raw = list(self.b.decode_batch(pts, self.slots))
        else:
            raw = [self.b.decode(pt, self.slots) for pt in pts]
        vals = [(v - off) / g if off else v / g for v in raw]
        for pt in pts:
            self.b.free(pt)
        if lay.kind == "slot0":
            return np.array([v[0] for v in vals])
        if lay.kind == "rep":
            return np.concatenate([v[np.arange(lay.H) * lay.hS] for v in vals])[:lay.count]
        idx = lay.slots_of_valid()
        return np.stack([v[idx] for v in vals]).reshape(lay.C, lay.H, lay.W)

    # ---- rotation key policy ----------------------------------------------------
    def _pow2_steps(self, k: int):
        """Signed power-of-two decomposition of a left rotation by k (non-adjacent form of k or
        of k - slots, whichever has fewer terms): left rotations by 2^i and right rotations by
        2^i (= left by slots - 2^i)."""
        def naf(v):
            out, i = [], 0
            while v:
                if v & 1:
                    d = 2 - (v & 3)          # +1 or -1
                    out.append(d << i)
                    v -= d
                v >>= 1
                i += 1
            return out
        k %= self.slots
        if k == 0:
            return []
        a, b = naf(k), naf(k - self.slots)
        best = a if len(a) <= len(b) else b
        return [x % self.slots for x in best]

    def _rot_many(self, cts, amounts):
        """[[rotLeft(ct, a) for a in amounts] for ct in cts]: exact keys -> hoisted batch (shared
        ModUps); pow2 keys -> each amount composed from power-of-two rotations, batched over cts."""
        if not cts or not amounts:
            return [[] for _ in cts]
        if self.rot_policy == "exact":
            if len(amounts) == 1:        # one amount: the fused K4 batch (no materialised ModUp)
                return [[h] for h in self.b.rot_left_batch(list(cts), amounts[0])]
            return self.b.rot_left_hoisted_batch(list(cts), amounts)
        out = [[None] * len(amounts) for _ in cts]
        for ai, a in enumerate(amounts):
            cur, own = list(cts), False
            steps = self._pow2_steps(a)
            if not steps:
                cur = [self.b.copy(h) for h in cts]
            for st in steps:
                nxt = self.b.rot_left_batch(cur, st)
                if own:
                    self._free_all(cur)
                cur, own = nxt, True
            for i, h in enumerate(cur):
                out[i][ai] = h
        return out

    # ---- helpers --------------------------------------------------------------------------
    def _plaintext(self, key, values_fn, level):
        """Weight / mask plaintexts at scale q_top (A8), encoded once per model (cached)."""
        pt = self._pts.get((key, level))
        if pt is None:
            pt = self.b.encode(values_fn(), float(self.q[level]), level)
            self._pts[(key, level)] = pt
        return pt

    def _free_all(self, hs, keep=()):
        keep = set(keep)
        for h in hs:
            if h not in keep:
                self.b.free(h)

    def _level(self, h):
        return self.b.ct_info(h)[0]

    # ---- layers ---------------------------------------------------------------------------
    def mask(self, cts, lay, li):
        """Zero the invalid slots before a padded conv: mulPlain by the 0/1 mask,
        rescale.  One level."""
        idx = lay.slots_of_valid()

        def vals():
            v = np.zeros(self.slots)
            v[idx] = 1.0
            return v
        pts = [self._plaintext(("mask", li), vals, self._level(ct)) for ct in cts]
        if hasattr(self.b, "mul_plain_batch"):   # one launch for the layer's channels
            ms = self.b.mul_plain_batch(list(cts), pts)
        else:
            ms = [self.b.mul_plain(ct, pt) for ct, pt in zip(cts, pts)]
        out = self.b.rescale_batch(ms)
        self._free_all(ms)
        return out, replace(lay, clean=True)

    @staticmethod
    def chw_geometry(lay, k, p, slots):
        """CHW tiling of a stride-1 conv input (NEXT-1): channel block stride CS (a power of two
        holding the plane plus the SAME padding on both sides), channels per ciphertext G, data
        offset of a channel inside its block."""
        pad_off = p * lay.hS + p * lay.wS
        span = (lay.H - 1) * lay.hS + (lay.W - 1) * lay.wS + 1
        cs = 1 << math.ceil(math.log2(span + 2 * pad_off))
        return cs, max(1, slots // cs), pad_off

    def _pack(self, cts, lay, cs, G, pad_off):
        """CHW packing (NEXT-1): clean channel c -> packed ciphertext c // G, block c % G,
        its data origin moved to block offset g cs + pad_off (one right rotation per channel
        outside block 0, batched per block; adds in between)."""
        C = lay.C
        npk = -(-C // G)
        packed = [None] * npk
        for g in range(G):
            chans = [c for c in range(g, C, G)]
            if not chans:
                continue
            shift = (g * cs + pad_off - lay.origin) % self.slots
            amt = (self.slots - shift) % self.slots
            if amt:
                rs = [r[0] for r in self._rot_many([cts[c] for c in chans], [amt])]
            else:
                rs = [self.b.copy(cts[c]) for c in chans]
            for c, r in zip(chans, rs):
                kk = c // G
                if packed[kk] is None:
                    packed[kk] = r
                else:
                    nxt = self.b.add(packed[kk], r)
                    self._free_all([packed[kk], r])
                    packed[kk] = nxt
        return packed

    @staticmethod
    def fc_chw_geometry(lay, slots):
        """CHW FC packing (NEXT-1): block stride cs = the plane's span rounded up to a power of
        two, G = channels per ciphertext (a power of two, <= slots / cs, no more than needed)."""
        span = (lay.H - 1) * lay.hS + (lay.W - 1) * lay.wS + 1
        cs = 1 << math.ceil(math.log2(span))
        G = min(max(1, slots // cs), 1 << math.ceil(math.log2(max(1, lay.C))))
        return cs, G

    def fc_chw(self, cts, lay, layer, w, beta, li):
        """CHW-tiled matmul (NEXT-1: the paper's "CHW-fc" layouts, P:722-725 with P:728): the
        (masked, clean) channels packed G per ciphertext at block stride cs, one mulPlain per
        (neuron, packed ciphertext) -- C / G instead of C -- with the weights laid on each block,
        one rescale, then log2(G cs) rotate-and-sum steps into slot 0 (the dot product over all
        blocks).  R = 1 form; the output is one ciphertext per neuron (slot-0 layout)."""
        if self.world > 1:
            raise NotImplementedError("CHW FC is single-GPU in this build")
        n_out = layer[1]
        masked = False
        if not lay.clean:
            cts, lay = self.mask(cts, lay, li)
            masked = True
        cs, G = self.fc_chw_geometry(lay, self.slots)
        packed = self._pack(cts, lay, cs, G, 0)
        if masked:
            self._free_all(cts)
        rel = lay.slots_of_valid() - lay.origin
        hw = lay.H * lay.W

        def vals(jo, kk):
            v = np.zeros(self.slots)
            for g in range(G):
                c = kk * G + g
                if c < lay.C:
                    v[g * cs + rel] = w[jo, c * hw:(c + 1) * hw]
            return v
        sums = self._mulplain_sums(packed, range(n_out), "fcchw", li, vals)
        self._free_all(packed)
        res = self.b.rescale_batch(sums)
        self._free_all(sums)
        res = self._rotate_sum(res, [1 << t for t in range(int(math.log2(G * cs)))])
        return self._bias(res, beta), Layout("slot0", n_out)

    def conv_chw(self, cts, lay, layer, w, beta, li):
        """CHW-tiled conv2d (NEXT-1), stride 1: G channels packed per ciphertext at
        block stride CS; the K^2 - 1 tap rotations are hoisted per PACKED ciphertext (G channels
        per key switch); per output channel one mulPlain per (packed ciphertext, tap) with the
        tap's weights laid on each channel block (the "mulv is required" of P:722), one rescale,
        then log2 G rotate-and-sum steps across blocks ("2 log(C) rotations"); the output
        channel lands in block 0 (HW layout, origin = the block data offset)."""
        _, oc_n, k, st, p = layer[:5]
        if st != 1:
            raise ValueError("CHW conv lowering supports stride 1")
        if self.world > 1:
            raise NotImplementedError("CHW conv is single-GPU in this build")
        if not lay.clean:
            cts, lay = self.mask(cts, lay, li)
            masked = True
        else:
            masked = False
        C = lay.C
        cs, G, pad_off = self.chw_geometry(lay, k, p, self.slots)
        npk = -(-C // G)
        packed = self._pack(cts, lay, cs, G, pad_off)
        if masked:
            self._free_all(cts)
        taps = [(i, j) for i in range(k) for j in range(k)]
        amounts = [((i - p) * lay.hS + (j - p) * lay.wS) % self.slots for i, j in taps]
        nz = [a for a in amounts if a]
        rot_all = self._rot_many(packed, nz)
        inputs, temps = [], []
        for x, rl in zip(packed, rot_all):
            it = iter(rl)
            for a in amounts:
                h = next(it) if a else x
                inputs.append(h)
                if a:
                    temps.append(h)
        lv = self._level(packed[0])
        rel = lay.slots_of_valid() - lay.origin       # plane positions relative to the data origin

        def vals(oc, kk, t):
            i, j = taps[t]
            v = np.zeros(self.slots)
            for g in range(G):
                c = kk * G + g
                if c < C:
                    v[g * cs + pad_off + rel] = w[oc, c, i, j]
            return v
        keys = [(("chw", li, oc, kk, t), lv) for oc in range(oc_n) for kk in range(npk) for t in range(len(taps))]
        todo = [(key, oc, kk, t) for key, (oc, kk, t) in
                zip(keys, [(oc, kk, t) for oc in range(oc_n) for kk in range(npk) for t in range(len(taps))])
                if key not in self._pts]
        for c0 in range(0, len(todo), 256):          # weight plaintexts, once per model, in batches
            chunk = todo[c0:c0 + 256]
            hs = self.b.encode_batch(np.stack([vals(oc, kk, t) for _k, oc, kk, t in chunk]), float(self.q[lv]), lv)
            for (key, _o, _kk, _t), h in zip(chunk, hs):
                self._pts[key] = h
        sums = self.b.mul_plain_accumulate(inputs, [self._pts[key] for key in keys], oc_n)
        self._free_all(temps + packed)
        res = self.b.rescale_batch(sums)
        self._free_all(sums)
        res = self._rotate_sum(res, [cs << t for t in range(int(math.log2(G)))])
        res = self._bias(res, beta)
        return res, Layout("hw", oc_n, lay.H, lay.W, lay.hS, lay.wS, pad_off, False)

    def conv(self, cts, lay, layer, w, beta, li):
        """Alg. 1: hoisted rotations per input channel + fused accumulation."""
        if len(layer) > 5 and layer[5] == "chw":
            return self.conv_chw(cts, lay, layer, w, beta, li)
        _, oc_n, k, st, p = layer[:5]
        own_in = self.owned(lay.C)
        if p > 0 and not lay.clean:
            cts, lay = self.mask(cts, lay, li)
            masked = True
        else:
            masked = False
        oc_part = self.sharded and self.partition == "oc"
        if oc_part:                               # north-star baseline: every rank holds all inputs
            gathered = self._gather(cts, lay.C)
            if masked:
                self._free_all(cts)
            cts, own_in, masked = gathered, range(lay.C), True
        amounts = [(lay.origin + (i - p) * lay.hS + (j - p) * lay.wS) % self.slots
                   for i in range(k) for j in range(k)]
        nz = [a for a in amounts if a]
        rotated, wcols, temps = [], [], []
        # every owned input channel x every non-zero tap: ModUps batched over channels, each key
        # word streamed once per group of channels (hisa_rot_left_hoisted_batch)
        allr = self._rot_many(list(cts), nz) if (nz and cts) else [[] for _ in cts]
        for ci, ct, rl in zip(own_in, cts, allr):
            rs = iter(rl)
            for a in amounts:                     # tap with amount 0 = the input itself
                h = next(rs) if a else ct
                rotated.append(h)
                if a:
                    temps.append(h)
            wcols.append(w[:, ci].reshape(oc_n, k * k))
        wmat = np.concatenate(wcols, axis=1) if wcols else np.zeros((oc_n, 0))
        if oc_part:
            own_out = self.owned(oc_n)
            outs = self._accumulate_local(rotated, wmat[own_out.start:own_out.stop])
        else:
            outs = self._accumulate(rotated, wmat, oc_n)
        self._free_all(temps)
        if masked:
            self._free_all(cts)
        res = self.b.rescale_batch(outs)
        self._free_all(outs)
        res = self._bias(res, beta)
        nl = Layout("hw", oc_n, (lay.H + 2 * p - k) // st + 1, (lay.W + 2 * p - k) // st + 1,
                    lay.hS * st, lay.wS * st, 0, False)
        return res, nl

    def _gather(self, cts, n: int):
        """All n channels of a sharded layer on every rank (NCCL all-gather); fresh
        handles (the caller frees them).  Single GPU: copies."""
        if not self.sharded:
            return [self.b.copy(h) for h in cts]
        from . import parallel
        return parallel.gather_outputs(self, cts, n)

    def _accumulate_local(self, rotated, wmat):
        """sum_t W[o, t] rotated[t] for the rows of wmat, on this rank alone (no exchange)."""
        if wmat.shape[0] == 0 or not rotated:
            return []
        return self.b.conv_accumulate(rotated, np.ascontiguousarray(wmat).ravel())

    def _accumulate(self, rotated, wmat, n_out):
        """sum_t W[o, t] rotated[t] for o < n_out (pre-rescale).  Single GPU: one fused kernel.
        Multi-GPU: partial sums over this rank's inputs for ALL outputs, NCCL reduce-scatter,
        mod-q fix-up; returns the outputs this rank owns (owned(n_out))."""
        if not self.sharded:
            return self.b.conv_accumulate(rotated, wmat.ravel())
        from . import parallel
        return parallel.reduce_scatter_partials(self, rotated, wmat, n_out)

    def act(self, cts, lay, square_only=False):
        """(A25) x'^2 + gamma: tensor + relinearize + rescale (+ addScalar): one level.
        gamma is this activation's (gain-scaled, A41) constant, in execution order."""
        sq = self.b.mul_batch(list(cts), list(cts))       # tensor + relin, batched
        out = self.b.rescale_batch(sq)
        self._free_all(sq)
        gamma = 0.0
        if not square_only:
            gamma = self.gammas[self._act_i]
            self._act_i += 1
        if gamma:
            out2 = [self.b.add_scalar(r, gamma) for r in out]
            self._free_all(out)
            out = out2
        return out, replace(lay, clean=False)

    def avgpool(self, cts, lay):
        """2x2 average pool (A26): x + rot(wS) + rot(hS) + rot(hS + wS), hoisted."""
        out = []
        allr = self._rot_many(list(cts), [lay.wS, lay.hS, lay.hS + lay.wS]) if cts else []
        for ct, r in zip(cts, allr):
            s1 = self.b.add(ct, r[0])
            s2 = self.b.add(r[1], r[2])
            out.append(self.b.add(s1, s2))
            self._free_all(r + [s1, s2])
        return out, Layout("hw", lay.C, lay.H // 2, lay.W // 2, lay.hS * 2, lay.wS * 2, lay.origin, False)

    def fire(self, cts, lay, layer, folded3, li):
        """SqueezeNet fire module (config 5, A33): squeeze 1x1 conv + act, mask (the 3x3 expand
        needs zeros around the valid plane), then ONE expand conv whose OC = e1 + e3
        outputs are the 1x1 expand (its weights at the centre tap of a 3x3 kernel, amount 0 = no
        rotation) and the 3x3 SAME expand -- the concatenation is the channel order -- + act."""
        _, sq, e1, e3 = layer
        (wsq, bsq), (we1, b1), (we3, b3) = folded3
        s, lay_s = self.conv(cts, lay, ("conv", sq, 1, 1, 0), wsq, bsq, (li, "sq"))
        s2, lay_s = self.act(s, lay_s)
        self._free_all(s)
        m, lay_m = self.mask(s2, lay_s, (li, "mask"))
        self._free_all(s2)
        wexp = np.zeros((e1 + e3, sq, 3, 3))
        wexp[:e1, :, 1, 1] = we1[:, :, 0, 0]
        wexp[e1:] = we3
        assert b1 == b3
        e, lay_e = self.conv(m, lay_m, ("conv", e1 + e3, 3, 1, 1), wexp, b1, (li, "exp"))
        self._free_all(m)
        out, lay_o = self.act(e, lay_e)
        self._free_all(e)
        return out, lay_o

    def gap(self, cts, lay):
        """Global average pool (A26): rotate-and-sum over the valid H x W grid (powers of two)
        into slot 0; the 1/(H W) is folded into the preceding linear layer."""
        if lay.H & (lay.H - 1) or lay.W & (lay.W - 1):
            raise ValueError("global average pool needs power-of-two H, W")
        amts = [lay.wS << t for t in range(int(math.log2(lay.W)))] + \
               [lay.hS << t for t in range(int(math.log2(lay.H)))]
        res = self._rotate_sum(list(cts), amts, consume=False) if amts else [self.b.copy(h) for h in cts]
        return res, Layout("slot0", lay.C)

    def _rotate_sum(self, res, amounts, consume=True):
        """acc += rot(acc, a) for a in amounts, every ciphertext under one key per step.  The
        input handles are freed unless consume=False (or amounts is empty)."""
        first = True
        for a in amounts:
            steps = self._pow2_steps(a) if self.rot_policy == "pow2" else [a]
            if len(steps) == 1:
                nxt = self.b.rot_add_batch(res, steps[0])   # x + rot(x, a), add fused into the permutation
            else:
                r = self._rot_many(res, [a])
                nxt = [self.b.add(x, rr[0]) for x, rr in zip(res, r)]
                self._free_all([rr[0] for rr in r])
            if consume or not first:
                self._free_all(res)
            res, first = nxt, False
        return res

    def _mulplain_sums(self, cts, rows, key, li, vals_fn):
        """acc_j = sum_c mulPlain(cts[c], P_{j,c}) for j in `rows` over ALL input channels c
        (cts = every input, gathered on every rank under a process group); P built by
        vals_fn(j, c).  One fused mulPlain-accumulate launch (hisa_mul_plain_accumulate)."""
        if not cts or len(rows) == 0:
            return []
        lv = self._level(cts[0])
        n_in = len(cts)
        keys = [((key, li, jo, ci), lv) for jo in rows for ci in range(n_in)]
        missing = [(k, jo, ci) for k, (jo, ci) in zip(keys, [(jo, ci) for jo in rows for ci in range(n_in)])
                   if k not in self._pts]
        if missing:   # the layer's weight plaintexts, encoded once per model in one batch
            hs = self.b.encode_batch(np.stack([vals_fn(jo, ci) for _k, jo, ci in missing]), float(self.q[lv]), lv)
            for (k, _jo, _ci), h in zip(missing, hs):
                self._pts[k] = h
        pts = [self._pts[k] for k in keys]
        return self.b.mul_plain_accumulate(list(cts), pts, len(rows))

    def _fc_inputs(self, cts, n: int):
        """SURVEY 8e FC plan: the FC's inputs all-gathered to every rank (returns (all inputs,
        temporaries to free)); single GPU: the inputs themselves."""
        if not self.sharded:
            return list(cts), []
        allc = self._gather(cts, n)
        return allc, allc

    def fc_replicated(self, cts, lay, layer, w, beta, li):
        """FC with R replicas per ciphertext ("replicas ... added in log number of
        rotations", A27): mask, replicate R times at block stride Bk (log2 R rotations), one
        mulPlain per (group of R neurons, input channel), rescale, rotate-and-sum inside each
        block; neuron g R + r ends in slot r Bk of ciphertext g.  Multi-GPU (8e): inputs
        all-gathered, the R-groups partitioned."""
        n_out, R = layer[1], layer[2]
        masked = []
        if not lay.clean:                          # each rank masks its own channels, then gathers
            masked, lay = self.mask(cts, lay, li)
            cts = masked
        cts, temp_in = self._fc_inputs(cts, lay.C)
        if temp_in:
            self._free_all(masked)
        else:
            temp_in = masked
        Bk = 1 << math.ceil(math.log2(lay.span()))
        if R * Bk > self.slots or R & (R - 1):
            raise ValueError(f"replicas R={R} x block {Bk} exceed {self.slots} slots")
        reps, temp = list(cts), bool(temp_in)
        for t in range(int(math.log2(R))):           # copies at r * Bk (right rotations)
            rs = [r[0] for r in self._rot_many(reps, [self.slots - (Bk << t)])]
            nxt = [self.b.add(x, r) for x, r in zip(reps, rs)]
            self._free_all(rs + (reps if temp else []))
            reps, temp = nxt, True
        idx = lay.slots_of_valid()
        hw = lay.H * lay.W
        n_groups = -(-n_out // R)

        def vals(g, c):
            v = np.zeros(self.slots)
            for r in range(R):
                j = g * R + r
                if j < n_out:
                    v[r * Bk + idx] = w[j, c * hw:(c + 1) * hw]
            return v
        sums = self._mulplain_sums(reps, self.owned(n_groups), "fcrep", li, vals)
        if temp:
            self._free_all(reps)
        res = self.b.rescale_batch(sums)
        self._free_all(sums)
        res = self._rotate_sum(res, [1 << t for t in range(int(math.log2(Bk)))])
        return self._bias(res, beta), Layout("rep", n_groups, H=R, hS=Bk, count=n_out)

    def fc_from_rep(self, cts, lay, layer, w, beta, li):
        """FC whose input holds R values per ciphertext at slots r * Bk: one mulPlain per
        (output, input ciphertext) with the weights at those slots, rescale, rotate-and-sum
        across the R blocks (log2 R rotations) into slot 0.  Multi-GPU: inputs all-gathered,
        outputs partitioned (8e)."""
        n_out = layer[1]
        R, Bk = lay.H, lay.hS
        cts, temp_in = self._fc_inputs(cts, lay.C)

        def vals(k, g):
            v = np.zeros(self.slots)
            for r in range(R):
                j = g * R + r
                if j < lay.count:
                    v[r * Bk] = w[k, j]
            return v
        sums = self._mulplain_sums(cts, self.owned(n_out), "fcfromrep", li, vals)
        self._free_all(temp_in)
        res = self.b.rescale_batch(sums)
        self._free_all(sums)
        res = self._rotate_sum(res, [Bk << t for t in range(int(math.log2(R)))])
        return self._bias(res, beta), Layout("slot0", n_out)

    def fc(self, cts, lay, layer, w, beta, li):
        """Matmul (A27): R = 1 (below), replicas (fc_replicated), or an input in
        replica layout (fc_from_rep).  Multi-GPU: the inputs are all-gathered and
        the output neurons partitioned across ranks -- no partial-sum exchange."""
        if lay.kind == "rep":
            return self.fc_from_rep(cts, lay, layer, w, beta, li)
        if lay.kind == "hw" and len(layer) > 3 and layer[3] == "chw":
            return self.fc_chw(cts, lay, layer, w, beta, li)
        if lay.kind == "hw" and len(layer) > 2 and layer[2] > 1:
            return self.fc_replicated(cts, lay, layer, w, beta, li)
        n_out = layer[1]
        own_out = self.owned(n_out)
        allc, temp_in = self._fc_inputs(cts, lay.C)
        if lay.kind == "slot0":          # next FC reads slot 0: scalar MACs, fused
            outs = self._accumulate_local(allc, w[own_out.start:own_out.stop, :])
            self._free_all(temp_in)
            res = self.b.rescale_batch(outs)
            self._free_all(outs)
            return self._bias(res, beta), Layout("slot0", n_out)
        idx = lay.slots_of_valid()
        hw = lay.H * lay.W
        steps = math.ceil(math.log2(lay.span()))

        def vals(jo, ci):
            v = np.zeros(self.slots)
            v[idx] = w[jo, ci * hw:(ci + 1) * hw]
            return v
        sums = self._mulplain_sums(allc, own_out, "fc", li, vals)
        self._free_all(temp_in)
        res = self.b.rescale_batch(sums)
        self._free_all(sums)
        res = self._rotate_sum(res, [1 << t for t in range(steps)])   # slot 0 <- dot product
        return self._bias(res, beta), Layout("slot0", n_out)

    def _bias(self, cts, beta):
        if not beta:
            return cts
        out = [self.b.add_scalar(h, beta) for h in cts]
        self._free_all(cts)
        return out

    # ---- forward ----------------------------------------------------------------------------
    def forward(self, cts, lay, trace=None):
        """Server-side evaluation of the whole network.  With a process group, `cts` are this
        rank's owned input channels and the result is this rank's owned output channels.
        `trace(layer_index, cts, layout)` (optional) is called after every layer, before the
        layer's inputs are freed (per-layer parity checks)."""
        wi = 0
        self._act_i = 0
        cur = list(cts)
        for li, layer in enumerate(self.net["layers"]):
            kind = layer[0]
            if kind in ("conv", "fc"):
                w, beta = self.folded[wi]
                wi += 1
                fn = self.conv if kind == "conv" else self.fc
                nxt, lay = fn(cur, lay, layer, w, beta, li)
            elif kind == "act":
                nxt, lay = self.act(cur, lay)
            elif kind == "square":
                nxt, lay = self.act(cur, lay, square_only=True)
            elif kind == "avgpool":
                nxt, lay = self.avgpool(cur, lay)
            elif kind == "fire":
                nxt, lay = self.fire(cur, lay, layer, self.folded[wi:wi + 3], li)
                wi += 3
            elif kind == "gap":
                nxt, lay = self.gap(cur, lay)
            else:
                raise ValueError(kind)
            self._free_all(cur, keep=cts)
            cur = nxt
            if trace is not None:
                trace(li, cur, lay)
        return cur, lay

    def forward_gathered(self, cts, lay):
        """forward() followed, under a process group, by the final all-gather: every rank ends
        with all output ciphertexts (rank 0 decrypts)."""
        out, lay = self.forward(cts, lay)
        if self.sharded:
            from . import parallel
            allc = parallel.gather_outputs(self, out, lay.C)
            self._free_all(out)
            out = allc
        return out, lay

    def shard_input(self, cts):
        """This rank's owned input channels of a full list (the rest are freed)."""
        own = self.owned(len(cts))
        mine = [cts[i] for i in own]
        self._free_all([h for i, h in enumerate(cts) if i not in own])
        return mine
