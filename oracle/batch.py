"""O-2: Baton's batch state machine, paper-literal (TEST INFRASTRUCTURE ONLY).

The three variables of P:L87 ("input_token, attention_mask, and KV_Cache") are
kept exactly as the paper manipulates them, as DENSE tensors whose shared
sequence axis grows and shrinks:

* ``mask``  -- attention_mask, uint8 [B][S], 1 = real token, 0 = padding or
               placeholder.
* ``K, V``  -- KV_Cache [layer][batch][head][seq][embed], float64 holding
               the exact bf16 values (reading C12).  Only ``seq`` (= S) changes.
* ``pad``   -- per-query ``index``, "which marks the end of the padding"
               (P:L124), i.e. the column where the query's live region begins.
* ``qid``   -- which query occupies each row (-1 = empty; reading C6).

Placeholders: the paper writes -inf into placeholder K/V cells.
Reading C2: they are don't-care cells, hidden by mask 0; the oracle writes the
``fill`` value (0.0 by default, NaN in the inertness pins) and never multiplies a
masked cell, so any fill is inert.

Operations (each cites the passage it follows):

* ``step``     P:L96  append one mask column (1 for live rows) and one KV column,
               then masked attention for every live row (via O-1 on the
               row's live columns gathered in ascending order).
* ``shape_step`` P:L101-113 the vector-SHAPING iteration (Baton without P&D):
               raw queries join with their whole prompt, every row's input is
               padded to the common width W (reading C4: mask and KV grow by W).
* ``insert``   P:L137 vector embedding: case l_q <= S end-aligned, front S-l_q
               placeholders; case l_q > S expand every row on the LEFT by l_q-S
               (KV fill, mask 0 for existing rows, 1 for the new query).
* ``remove``   P:L105 zero the finished query's mask row; P:L107 its KV becomes
               placeholder (fill).
* ``release``  P:L123-124 drop the [0 : min(index_i)] front segment of KV and mask.
* ``extract``  P:L144 "temporarily store the Keys and Values" of a query (its live
               region, reading C16) -- the caller then removes it.
* ``compact``  P:L147 batch-size scaling: move queries out of the released slot
               range (reading C19: stable, lowest free slot, ascending).
"""
import numpy as np

from .attention import solo_attention


class OracleError(Exception):
    pass


class SlotBusy(OracleError):
    pass


class SlotEmpty(OracleError):
    pass


class Capacity(OracleError):
    pass


class Shard:
    def __init__(self, B, L, H_q, H_kv, D, S_cap, fill=0.0, kv=True):
        self.B, self.L, self.H_q, self.H_kv, self.D, self.S_cap = B, L, H_q, H_kv, D, S_cap
        self.fill = fill
        self.kv = kv
        self.S = 0
        self.mask = np.zeros((B, 0), dtype=np.uint8)
        self.pad = np.zeros(B, dtype=np.int64)
        self.qid = np.full(B, -1, dtype=np.int64)
        if kv:
            self.K = np.zeros((L, B, H_kv, 0, D), dtype=np.float64)
            self.V = np.zeros((L, B, H_kv, 0, D), dtype=np.float64)

    # ------------------------------------------------------------------ queries
    def occupied(self):
        return [b for b in range(self.B) if self.qid[b] >= 0]

    def lens(self):
        """Live length of every row: the number of mask-1 columns."""
        return self.mask.sum(axis=1, dtype=np.int64) if self.S else np.zeros(self.B, np.int64)

    # ------------------------------------------------------------------ P:L137
    def insert(self, slot, qid, l_q, K_pref=None, V_pref=None):
        """Embed a prefilled query (its K/V of length l_q) into row ``slot``."""
        if self.qid[slot] >= 0:
            raise SlotBusy(f"slot {slot} occupied")
        if l_q < 1 or l_q > self.S_cap:
            raise Capacity(f"l_q={l_q}")
        if self.kv:
            K_pref = np.asarray(K_pref, dtype=np.float64)
            V_pref = np.asarray(V_pref, dtype=np.float64)
            assert K_pref.shape == (self.L, self.H_kv, l_q, self.D)
        S = self.S
        if l_q <= S:
            # case 1: "embedded into KV_Cache in an end-aligned manner, and the
            # remaining front part ... with length l_kv - l_q, will be filled"
            p = S - l_q
            self.mask[slot, :] = 0
            self.mask[slot, p:] = 1
            if self.kv:
                self.K[:, slot, :, :p, :] = self.fill
                self.V[:, slot, :, :p, :] = self.fill
                self.K[:, slot, :, p:, :] = K_pref
                self.V[:, slot, :, p:, :] = V_pref
            self.pad[slot] = p
        else:
            # case 2: "the length of l_q - l_kv should be added to the left side
            # of KV_Cache ... The expansions of existing queries will be filled
            # with 0, and ... the values of new query's attention_mask ... 1"
            e = l_q - S
            if l_q > self.S_cap:
                raise Capacity("expansion beyond capacity")
            self.mask = np.concatenate([np.zeros((self.B, e), np.uint8), self.mask], axis=1)
            if self.kv:
                padk = np.full((self.L, self.B, self.H_kv, e, self.D), self.fill)
                self.K = np.concatenate([padk, self.K], axis=3)
                self.V = np.concatenate([padk.copy(), self.V], axis=3)
            for b in self.occupied():
                self.pad[b] += e
            self.S = l_q
            self.mask[slot, :] = 1
            if self.kv:
                self.K[:, slot] = K_pref
                self.V[:, slot] = V_pref
            self.pad[slot] = 0
        self.qid[slot] = qid

    # ------------------------------------------------------------------ P:L96
    def step(self, q=None, k_new=None, v_new=None):
        """One decode iteration.

        q: [L][B][H_q][D]; k_new, v_new: [L][B][H_kv][D] (rows of empty slots are
        ignored).  Returns o: [L][B][H_q][D] with empty rows zeroed (reading C6),
        or None in metadata-only mode."""
        if self.S + 1 > self.S_cap:
            raise Capacity("S would exceed capacity")
        occ = self.qid >= 0
        col = occ.astype(np.uint8)[:, None]          # "a column with the value of all 1"
        self.mask = np.concatenate([self.mask, col], axis=1)
        self.S += 1
        if not self.kv:
            return None
        kc = np.full((self.L, self.B, self.H_kv, 1, self.D), self.fill)
        vc = np.full((self.L, self.B, self.H_kv, 1, self.D), self.fill)
        for b in np.nonzero(occ)[0]:
            kc[:, b, :, 0, :] = k_new[:, b]
            vc[:, b, :, 0, :] = v_new[:, b]
        # "appends the inter-relationships ... to KV_Cache"
        self.K = np.concatenate([self.K, kc], axis=3)
        self.V = np.concatenate([self.V, vc], axis=3)
        out = np.zeros((self.L, self.B, self.H_q, self.D), dtype=np.float64)
        for b in np.nonzero(occ)[0]:
            live = np.nonzero(self.mask[b])[0]       # masked columns never enter the sum
            for l in range(self.L):
                out[l, b] = solo_attention(q[l, b], self.K[l, b][:, live, :],
                                           self.V[l, b][:, live, :])
        return out

    # ------------------------------------------------------------------ P:L101-113
    def shape_step(self, new=(), q=None, k_new=None, v_new=None):
        """One iteration of the vector-SHAPING path (Baton without P&D, NEXT-1).

        ``new`` lists (slot, qid, l_q) raw queries inserted now: their rows must be
        empty (the finished query's row was removed: "set all the values of the
        query^2 part of the current attention_mask tensor to 0").  The
        input width is W = max(1, max l_q): "pad the latest token of query^0 and
        query^1 to the same length as query^3".
          * surviving rows append mask [1, 0^(W-1)] ("appended with values of 0
            according to the padding");
          * a new row appends "an all-1 vector with the same length of query^3"
            (P:L105), then 0^(W-l_q) if another insert is longer;
          * every row appends W KV columns (reading C4: mask and KV both grow by
            the input width); padding tokens' KV cells are placeholders (fill).
        Input token t of row b attends to the columns j with mask 1 and
        j <= S_old + t (the new query's prefill is causal within its block;
        a survivor's real token is t = 0, so it is an ordinary decode).

        q: [L][B][W][H_q][D]; k_new, v_new: [L][B][W][H_kv][D] (only real tokens
        are read).  Returns o: [L][B][W][H_q][D], zero on padding tokens and empty
        rows (their GPU rows are the bubble of P:L128), or None (metadata mode)."""
        new = [(int(s), int(qd), int(l)) for s, qd, l in new]
        W = max([1] + [l for _, _, l in new])
        if self.S + W > self.S_cap:
            raise Capacity("S would exceed capacity")
        for s, _, l in new:
            if self.qid[s] >= 0:
                raise SlotBusy(f"slot {s} occupied")
            if l < 1:
                raise Capacity(f"l_q={l}")
        S0 = self.S
        survivors = [b for b in range(self.B) if self.qid[b] >= 0]
        real = np.zeros((self.B, W), dtype=bool)          # real input tokens
        for b in survivors:
            real[b, 0] = True
        for s, qd, l in new:
            real[s, :l] = True
            self.qid[s] = qd
            self.pad[s] = S0                               # its live region starts here
        self.mask = np.concatenate([self.mask, real.astype(np.uint8)], axis=1)
        self.S = S0 + W
        if not self.kv:
            return None
        kc = np.full((self.L, self.B, self.H_kv, W, self.D), self.fill)
        vc = np.full((self.L, self.B, self.H_kv, W, self.D), self.fill)
        for b, t in zip(*np.nonzero(real)):
            kc[:, b, :, t, :] = k_new[:, b, t]
            vc[:, b, :, t, :] = v_new[:, b, t]
        self.K = np.concatenate([self.K, kc], axis=3)
        self.V = np.concatenate([self.V, vc], axis=3)
        out = np.zeros((self.L, self.B, W, self.H_q, self.D), dtype=np.float64)
        for b, t in zip(*np.nonzero(real)):
            live = np.nonzero(self.mask[b, :S0 + t + 1])[0]   # masked columns never enter
            for l in range(self.L):
                out[l, b, t] = solo_attention(q[l, b, t], self.K[l, b][:, live, :],
                                              self.V[l, b][:, live, :])
        return out

    # ------------------------------------------------------------------ P:L105-107
    def remove(self, slot):
        if self.qid[slot] < 0:
            raise SlotEmpty(f"slot {slot} empty")
        self.mask[slot, :] = 0                       # "set all the values ... to 0"
        if self.kv:
            self.K[:, slot] = self.fill              # placeholder (-inf in the paper, C2)
            self.V[:, slot] = self.fill
        self.qid[slot] = -1
        self.pad[slot] = 0

    # ------------------------------------------------------------------ P:L124
    def release(self):
        """Release the front [0 : min(index_i)] of KV_Cache and attention_mask."""
        occ = self.occupied()
        p = min(int(self.pad[b]) for b in occ) if occ else self.S
        if p:
            self.mask = self.mask[:, p:]
            if self.kv:
                self.K = self.K[:, :, :, p:, :]
                self.V = self.V[:, :, :, p:, :]
            for b in occ:
                self.pad[b] -= p
            self.S -= p
        return p

    # ------------------------------------------------------------------ P:L144
    def extract(self, slot):
        """The query's stored Keys/Values: its live region [index, S) (C16)."""
        if self.qid[slot] < 0:
            raise SlotEmpty(f"slot {slot} empty")
        p = int(self.pad[slot])
        if not self.kv:
            return None, None
        return (self.K[:, slot, :, p:, :].copy(), self.V[:, slot, :, p:, :].copy())

    # ------------------------------------------------------------------ P:L147
    def compact(self, n):
        """Move every query in rows >= n to the lowest free row < n (ascending).
        Returns old_to_new (identity for unmoved rows)."""
        old_to_new = list(range(self.B))
        for b in range(n, self.B):
            if self.qid[b] < 0:
                continue
            free = [f for f in range(n) if self.qid[f] < 0]
            if not free:
                raise Capacity("not enough free rows to compact")
            f = free[0]
            self.mask[f, :] = self.mask[b, :]
            self.mask[b, :] = 0
            if self.kv:
                self.K[:, f] = self.K[:, b]
                self.V[:, f] = self.V[:, b]
                self.K[:, b] = self.fill
                self.V[:, b] = self.fill
            self.pad[f], self.pad[b] = self.pad[b], 0
            self.qid[f], self.qid[b] = self.qid[b], -1
            old_to_new[b] = f
        return old_to_new

    # ------------------------------------------------------------------ views
    def snapshot(self):
        return {"S": self.S, "mask": self.mask.copy(), "pad": self.pad.copy(),
                "qid": self.qid.copy(), "lens": self.lens()}

    def live_kv(self, slot):
        """K/V of a row's live region in logical order (gathered by the mask)."""
        live = np.nonzero(self.mask[slot])[0]
        return self.K[:, slot][:, :, live, :], self.V[:, slot][:, :, live, :]
