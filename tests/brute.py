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


def automorphisms_backtrack(k, edges, cap=None):
    """|Aut(T)| of an (unrooted) tree by explicit enumeration: every bijection
    V_T -> V_T that maps edges to edges, built vertex by vertex in BFS
    order (each vertex after the first must land on a neighbour of its parent's
    image, degrees must match).  Independent of the AHU product formula.  Returns
    None if more than `cap` automorphisms exist (too many to list)."""
    adj = [set() for _ in range(k)]
    for a, b in edges:
        adj[a].add(b)
        adj[b].add(a)
    deg = [len(x) for x in adj]
    order, parent, seen = [0], {0: -1}, {0}
    i = 0
    while i < len(order):
        for w in sorted(adj[order[i]]):
            if w not in seen:
                seen.add(w)
                parent[w] = order[i]
                order.append(w)
        i += 1
    phi = [-1] * k
    used = [False] * k
    count = 0

    def rec(t):
        nonlocal count
        if cap is not None and count > cap:
            return
        if t == k:
            count += 1
            return
        v = order[t]
        cand = range(k) if parent[v] < 0 else adj[phi[parent[v]]]
        for x in cand:
            if used[x] or deg[x] != deg[v]:
                continue
            if any(phi[u] >= 0 and (phi[u] in adj[x]) != (u in adj[v]) for u in range(k)):
                continue
            phi[v] = x
            used[x] = True
            rec(t + 1)
            used[x] = False
            phi[v] = -1

    rec(0)
    return None if (cap is not None and count > cap) else count
