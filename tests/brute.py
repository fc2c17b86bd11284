"""Brute-force enumeration of (colourful) injective homomorphisms T -> G.

The pin the oracle is checked against (SURVEY §8(c) "What pins each part" 1):
it follows the DEFINITION, not the DP —
  colorful_j = #{φ: V_T -> V_G injective, (u,v)∈E_T ⇒ (φu,φv)∈E_G,
                 colours c_j(φ(u)) pairwise distinct}
  emb(T,G)   = #injective homomorphisms / α
Only for tiny inputs (n <= ~10, k <= ~6).
"""
from __future__ import annotations


def _adjsets(csr):
    ro, ci = csr.row_offsets, csr.col_indices
    return [set(int(x) for x in ci[ro[i]:ro[i + 1]]) for i in range(csr.n)]


def injective_homs(csr, k, edges, colors=None):
    """Number of injective homomorphisms (colourful ones only if colors given)."""
    adj = _adjsets(csr)
    tadj = [[] for _ in range(k)]
    for a, b in edges:
        tadj[a].append(b)
        tadj[b].append(a)
    # order template vertices so each (after the first) has an earlier neighbour
    order, seen = [0], {0}
    i = 0
    while i < len(order):
        for w in sorted(tadj[order[i]]):
            if w not in seen:
                seen.add(w)
                order.append(w)
        i += 1
    pos = {v: t for t, v in enumerate(order)}
    back = [[u for u in tadj[v] if pos[u] < pos[v]] for v in order]
    phi = [-1] * k
    used = set()
    used_col = set()
    total = 0

    def rec(t):
        nonlocal total
        if t == k:
            total += 1
            return
        v = order[t]
        if back[t]:
            cand = adj[phi[back[t][0]]]
        else:
            cand = range(csr.n)
        for x in cand:
            if x in used:
                continue
            if colors is not None and int(colors[x]) in used_col:
                continue
            if any(x not in adj[phi[u]] for u in back[t][1:]):
                continue
            phi[v] = x
            used.add(x)
            if colors is not None:
                used_col.add(int(colors[x]))
            rec(t + 1)
            used.discard(x)
            if colors is not None:
                used_col.discard(int(colors[x]))
            phi[v] = -1

    rec(0)
    return total
