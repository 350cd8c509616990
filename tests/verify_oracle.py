"""Pure-Python restatement of the reference's prefix-tree verification
(decode.cpp:32-43, 209-421) over the C oracle's forward (oracle/egt_oracle.c
egto_forward, model.cpp:118-202).  Test infrastructure only; small cases."""
from __future__ import annotations

import numpy as np


def children(trie, node):
    ch = [j for j in range(1, len(trie.token)) if trie.parent[j] == node]
    return sorted(ch, key=lambda j: int(trie.token[j]))


def restrict_row(row, trie, node):
    """restrict_row + log_softmax (decode.cpp:32-43, model.cpp:370-377):
    f32 max, partition sum in double over exp(f32(l - m)), f32 result."""
    ch = children(trie, node)
    vals = np.array([row[int(trie.token[c])] for c in ch], np.float32)
    m = np.float32(vals.max())
    d = (vals - m).astype(np.float32)
    z = float(np.sum(np.exp(d.astype(np.float64))))
    lz = np.float32(np.log(z))
    return ch, (d - lz).astype(np.float32)


def flatten_subtree(trie, beams):
    """decode.cpp:209-238: per beam, DFS over its node's strict descendants,
    children in ascending token order."""
    out = []
    for b, beam in enumerate(beams):
        stack = [(c, -1) for c in reversed(children(trie, beam.node))]
        while stack:
            node, parent = stack.pop()
            depth = 0 if parent < 0 else out[parent]["depth"] + 1
            out.append(dict(token=int(trie.token[node]), parent=parent, depth=depth, trie_node=node, beam=b))
            me = len(out) - 1
            for c in reversed(children(trie, node)):
                stack.append((c, me))
    return out


def build_tree_mask(flat, prompt, beams):
    """decode.cpp:240-299."""
    lens = [len(prompt) + len(b.tokens) for b in beams]
    lmax = max(lens)
    off = len(beams) * lmax
    R = off + len(flat)
    vis = np.zeros((R, R), bool)
    tokens = np.zeros(R, np.int32)
    pos = np.zeros(R, np.int32)
    for b, beam in enumerate(beams):
        seq = list(prompt) + list(beam.tokens)
        first = b * lmax + (lmax - len(seq))
        for j, t in enumerate(seq):
            tokens[first + j] = t
            pos[first + j] = j
            vis[first + j, first: first + j + 1] = True
    for f, fn in enumerate(flat):
        r = off + f
        tokens[r] = fn["token"]
        pos[r] = lens[fn["beam"]] + fn["depth"]
        first = fn["beam"] * lmax + (lmax - lens[fn["beam"]])
        vis[r, first: first + lens[fn["beam"]]] = True
        p = f
        while p >= 0:
            vis[r, off + p] = True
            p = flat[p]["parent"]
    return vis, tokens, pos, lmax, off


def is_leaf(trie, node):
    return not children(trie, node)


def verify_parallel(forward, trie, prompt, beams, beam_size):
    """decode.cpp:336-421 with `forward(tokens, positions, vis) -> logits`."""
    flat = flatten_subtree(trie, beams)
    vis, tokens, pos, lmax, off = build_tree_mask(flat, prompt, beams)
    logits = forward(tokens, pos, vis)
    seeds = {}
    for b, beam in enumerate(beams):
        if not is_leaf(trie, beam.node):
            seeds[b] = restrict_row(logits[b * lmax + lmax - 1], trie, beam.node)
    rows = {}
    for f, fn in enumerate(flat):
        if not is_leaf(trie, fn["trie_node"]):
            rows[f] = restrict_row(logits[off + f], trie, fn["trie_node"])
    scores = []
    for f, fn in enumerate(flat):  # accumulate_bscores (decode.cpp:301-334)
        if fn["parent"] < 0:
            ch, lp = seeds[fn["beam"]]
            base = beams[fn["beam"]].log_prob
        else:
            ch, lp = rows[fn["parent"]]
            base = scores[fn["parent"]]
        scores.append(base + float(lp[ch.index(fn["trie_node"])]))
    cands = [(beam.log_prob, b, -1) for b, beam in enumerate(beams) if is_leaf(trie, beam.node)]
    cands += [(scores[f], fn["beam"], f) for f, fn in enumerate(flat) if is_leaf(trie, fn["trie_node"])]
    cands.sort(key=lambda c: (-c[0], c[1], c[2]))
    out = []
    for score, b, f in cands[:beam_size]:
        toks = list(beams[b].tokens)
        if f < 0:
            payload = int(trie.payload[beams[b].node])
        else:
            path = []
            p = f
            while p >= 0:
                path.append(flat[p]["token"])
                p = flat[p]["parent"]
            toks += path[::-1]
            payload = int(trie.payload[flat[f]["trie_node"]])
        out.append({"tokens": toks, "score": score, "payload": payload, "beam": b})
    return out, {"flattened_nodes": len(flat), "rows": len(tokens)}
