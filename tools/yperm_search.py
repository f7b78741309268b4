"""Local search for the y-line assignment of the N = 4 FP64 tile (c_yperm_5x5 in
csrc/esdg_kernels.cuh): 125 threads, 125 y lines (element e of the CTA, x, z); a
thread may sweep any of them. Cost = shared-memory wavefronts of one CTA-wide access
to the node-value arrays (64-bit per half-warp, 128-bit per quarter-warp; word
index 125 e + x + 25 z) and to the slab (64-bit; 625 e + x + 25 z). Development
aid; prints the table."""
import random

T = 125
lines = [(e, x, z) for e in range(5) for z in range(5) for x in range(5)]


def groups(n):
    out = []
    for w in range(0, T, 32):
        lanes = list(range(w, min(w + 32, T)))
        out += [lanes[h:h + n] for h in range(0, 32, n) if lanes[h:h + n]]
    return out


H, Q = groups(16), groups(8)
node = lambda l: 125 * l[0] + l[1] + 25 * l[2]
slab = lambda l: 625 * l[0] + l[1] + 25 * l[2]


def worst(grp, a, f, m):
    cnt = {}
    for t in grp:
        r = f(a[t]) % m
        cnt[r] = cnt.get(r, 0) + 1
    return max(cnt.values())


def parts(a):
    return (sum(worst(g, a, node, 16) for g in H), sum(worst(g, a, node, 8) for g in Q),
            sum(worst(g, a, slab, 16) for g in H))


def cost(a):
    p = parts(a)
    return p[0] + p[1] + 2 * p[2]


print("natural assignment:", parts(lines), "ideal (8, 16, 8)")
random.seed(5)
cur = list(lines)
cc = best = cost(cur)
best_a = list(cur)
for _ in range(1500000):
    i, j = random.sample(range(T), 2)
    cur[i], cur[j] = cur[j], cur[i]
    c = cost(cur)
    if c <= cc:
        cc = c
        if c < best:
            best, best_a = c, list(cur)
    else:
        cur[i], cur[j] = cur[j], cur[i]
print("found:", parts(best_a))
print([l[0] * 25 + l[1] + 5 * l[2] for l in best_a])
