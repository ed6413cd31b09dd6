"""Batcher odd-even merge sort network for 32 inputs, pruned to 27 live inputs (inputs 27..31 are
+inf padding: a comparator whose upper wire is known to hold +inf is a no-op).  Verified here by the
0-1 principle on random inputs.  Prints the comparator list for lor_xh1.cu (k_xh1_sym)."""
import itertools
import random


def batcher(n):
    net = []
    p = 1
    while p < n:
        k = p
        while k >= 1:
            for j in range(k % p, n - k, 2 * k):
                for i in range(min(k, n - j - k)):
                    if (i + j) // (2 * p) == (i + j + k) // (2 * p):
                        net.append((i + j, i + j + k))
            k //= 2
        p *= 2
    return net


def prune(net, live):
    inf = [i >= live for i in range(32)]
    out = []
    for a, b in net:
        if inf[b]:
            continue
        out.append((a, b))
        inf[a], inf[b] = inf[a] and inf[b], inf[a] or inf[b]
    return out


net = prune(batcher(32), 27)
rng = random.Random(0)
for _ in range(20000):
    v = [rng.randrange(1000) for _ in range(27)] + [10 ** 9] * 5
    for a, b in net:
        if v[b] < v[a]:
            v[a], v[b] = v[b], v[a]
    assert v[:27] == sorted(v[:27])
print(len(net))
print(", ".join(f"{a * 32 + b}" for a, b in net))
