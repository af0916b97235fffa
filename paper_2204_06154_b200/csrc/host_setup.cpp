// Host-side setup of libmgm: Morton ordering, exact grid kNN, weighted sample elimination,
// greedy colouring, CSR transpose, dense LU.  Compiled with -O3 -ffp-contract=off so that
// every floating-point decision (distances, WSE weights) follows DESIGN.md's written rules
// bit for bit.  Citations: P:n = PAPER.md line n; O-numbers = DESIGN.md readings.
#include "mgm_internal.h"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <limits>
#include <thread>

namespace mgm {

template <class F>
static void parallel_for(i64 n, int nthreads, F&& f) {
    if (nthreads <= 1 || n < 4096) {
        f(0, n);
        return;
    }
    std::vector<std::thread> th;
    i64 chunk = (n + nthreads - 1) / nthreads;
    for (int t = 0; t < nthreads; ++t) {
        i64 b = t * chunk, e = std::min(n, b + chunk);
        if (b >= e) break;
        th.emplace_back([&f, b, e] { f(b, e); });
    }
    for (auto& x : th) x.join();
}

// ---------------------------------------------------------------------------------------
// O1: Morton order.  Quantise each axis with the common extent to 21 bits, interleave
// (x at bit 3b+2, y at 3b+1, z at 3b), sort by (key, index).
// ---------------------------------------------------------------------------------------
static inline uint64_t spread3(uint64_t v) {  // 21 bits -> every third bit
    v &= 0x1fffffull;
    v = (v | (v << 32)) & 0x1f00000000ffffull;
    v = (v | (v << 16)) & 0x1f0000ff0000ffull;
    v = (v | (v << 8)) & 0x100f00f00f00f00full;
    v = (v | (v << 4)) & 0x10c30c30c30c30c3ull;
    v = (v | (v << 2)) & 0x1249249249249249ull;
    return v;
}

bool morton_order(const double* pts, i64 n, std::vector<i64>& perm) {
    double lo[3], hi[3];
    for (int a = 0; a < 3; ++a) lo[a] = hi[a] = pts[a];
    for (i64 i = 0; i < n; ++i)
        for (int a = 0; a < 3; ++a) {
            lo[a] = std::min(lo[a], pts[3 * i + a]);
            hi[a] = std::max(hi[a], pts[3 * i + a]);
        }
    double ext = std::max(hi[0] - lo[0], std::max(hi[1] - lo[1], hi[2] - lo[2]));
    if (!(ext > 0.0)) return false;
    std::vector<std::pair<uint64_t, i64>> keys(n);
    for (i64 i = 0; i < n; ++i) {
        uint64_t q[3];
        for (int a = 0; a < 3; ++a) {
            double s = std::floor(((pts[3 * i + a] - lo[a]) / ext) * 2097152.0);
            i64 v = (i64)s;
            q[a] = (uint64_t)std::min<i64>(std::max<i64>(v, 0), 2097151);
        }
        keys[i] = {(spread3(q[0]) << 2) | (spread3(q[1]) << 1) | spread3(q[2]), i};
    }
    {  // chunks sorted on threads, then merged pairwise (keys are distinct: same order)
        const int T = n >= (1 << 18) ? std::max(1, std::min(16, (int)std::thread::hardware_concurrency())) : 1;
        std::vector<i64> b(T + 1);
        for (int t = 0; t <= T; ++t) b[t] = n * t / T;
        std::vector<std::thread> th;
        for (int t = 0; t < T; ++t) th.emplace_back([&, t] { std::sort(keys.begin() + b[t], keys.begin() + b[t + 1]); });
        for (auto& x : th) x.join();
        std::vector<std::pair<uint64_t, i64>> tmp(T > 1 ? n : 0);
        for (int w = 1; w < T; w *= 2) {
            th.clear();
            for (int t = 0; t < T; t += 2 * w)
                th.emplace_back([&, t] {
                    const i64 lo = b[t], mid = b[std::min(T, t + w)], hi = b[std::min(T, t + 2 * w)];
                    std::merge(keys.begin() + lo, keys.begin() + mid, keys.begin() + mid, keys.begin() + hi, tmp.begin() + lo);
                });
            for (auto& x : th) x.join();
            keys.swap(tmp);
        }
    }
    perm.resize(n);
    for (i64 i = 0; i < n; ++i) perm[i] = keys[i].second;
    return true;
}

// ---------------------------------------------------------------------------------------
// Uniform grid over a point set (cells sorted by linear id; dense cell table).
// ---------------------------------------------------------------------------------------
namespace {
struct Grid {
    double lo[3], cell;
    i64 dims[3];
    std::vector<i64> start;  // ncell + 1
    std::vector<i32> items;
    const double* pts;

    void build(const double* p, i64 n, double cell_size) {
        pts = p;
        for (int a = 0; a < 3; ++a) lo[a] = p[a];
        double hi[3] = {p[0], p[1], p[2]};
        for (i64 i = 0; i < n; ++i)
            for (int a = 0; a < 3; ++a) {
                lo[a] = std::min(lo[a], p[3 * i + a]);
                hi[a] = std::max(hi[a], p[3 * i + a]);
            }
        cell = cell_size;
        i64 total = 1;
        for (int a = 0; a < 3; ++a) {
            dims[a] = std::max<i64>(1, (i64)std::floor((hi[a] - lo[a]) / cell) + 1);
            total *= dims[a];
        }
        // keep the dense table bounded (cells only grow, so correctness is unaffected)
        while (total > 4 * n + 64) {
            cell *= 1.26;
            total = 1;
            for (int a = 0; a < 3; ++a) {
                dims[a] = std::max<i64>(1, (i64)std::floor((hi[a] - lo[a]) / cell) + 1);
                total *= dims[a];
            }
        }
        start.assign(total + 1, 0);
        std::vector<i64> cid(n);
        for (i64 i = 0; i < n; ++i) {
            cid[i] = cell_of(p + 3 * i);
            start[cid[i] + 1]++;
        }
        for (i64 c = 0; c < total; ++c) start[c + 1] += start[c];
        items.resize(n);
        std::vector<i64> fill(start.begin(), start.end() - 1);
        for (i64 i = 0; i < n; ++i) items[fill[cid[i]]++] = (i32)i;
    }
    void coords(const double* x, i64* c) const {
        for (int a = 0; a < 3; ++a) {
            i64 v = (i64)std::floor((x[a] - lo[a]) / cell);
            c[a] = std::min<i64>(std::max<i64>(v, 0), dims[a] - 1);
        }
    }
    i64 cell_of(const double* x) const {
        i64 c[3];
        coords(x, c);
        return (c[2] * dims[1] + c[1]) * dims[0] + c[0];
    }
};

// O2 squared distance: dx = y - x; (dx*dx + dy*dy) + dz*dz, no FMA (-ffp-contract=off).
inline double dist2(const double* x, const double* y) {
    double dx = y[0] - x[0], dy = y[1] - x[1], dz = y[2] - x[2];
    double s = dx * dx + dy * dy;
    return s + dz * dz;
}

struct KBest {
    int k;
    double* d;
    i32* j;
    int count = 0;
    void reset() { count = 0; }
    bool full() const { return count == k; }
    // insert keeping ascending (d, j)
    void offer(double dd, i32 jj) {
        if (count == k && (dd > d[k - 1] || (dd == d[k - 1] && jj > j[k - 1]))) return;
        int p = (count < k) ? count++ : k - 1;
        while (p > 0 && (d[p - 1] > dd || (d[p - 1] == dd && j[p - 1] > jj))) {
            d[p] = d[p - 1];
            j[p] = j[p - 1];
            --p;
        }
        d[p] = dd;
        j[p] = jj;
    }
};

double default_cell(const double* p, i64 n, int k) {
    double lo[3] = {p[0], p[1], p[2]}, hi[3] = {p[0], p[1], p[2]};
    for (i64 i = 0; i < n; ++i)
        for (int a = 0; a < 3; ++a) {
            lo[a] = std::min(lo[a], p[3 * i + a]);
            hi[a] = std::max(hi[a], p[3 * i + a]);
        }
    double ext = std::max(hi[0] - lo[0], std::max(hi[1] - lo[1], hi[2] - lo[2]));
    double vol = 1.0;
    for (int a = 0; a < 3; ++a) vol *= std::max(hi[a] - lo[a], 1e-3 * ext);
    double c = std::cbrt(vol * std::max(1, k / 4) / (double)n);
    return c > 0 ? c : 1.0;
}
}  // namespace

// Exact kNN by expanding Chebyshev shells of grid cells; stops when the k-th best squared
// distance is strictly below the squared distance to every unvisited cell.
void knn_grid(const double* pts, i64 n, const double* qry, i64 nq, int k, std::vector<i32>& out,
              int nthreads) {
    out.assign((size_t)nq * k, -1);
    Grid g;
    g.build(pts, n, default_cell(pts, n, k));
    {  // surface clouds fill few cells of the box: shrink the cells towards ~k/2 points per
       // occupied cell (the result does not depend on the cell size)
        i64 occ = 0;
        for (size_t c = 0; c + 1 < g.start.size(); ++c) occ += g.start[c + 1] > g.start[c];
        const double per = (double)n / (double)std::max<i64>(occ, 1);
        if (per > 2.0 * k) g.build(pts, n, g.cell * std::sqrt(0.5 * k / per));
    }
    parallel_for(nq, nthreads, [&](i64 b, i64 e) {
        std::vector<double> bd(k);
        std::vector<i32> bj(k);
        KBest best{k, bd.data(), bj.data()};
        for (i64 q = b; q < e; ++q) {
            const double* x = qry + 3 * q;
            best.reset();
            i64 c[3];
            g.coords(x, c);
            i64 maxr = std::max(g.dims[0], std::max(g.dims[1], g.dims[2]));
            for (i64 r = 0; r <= maxr; ++r) {
                for (i64 z = c[2] - r; z <= c[2] + r; ++z) {
                    if (z < 0 || z >= g.dims[2]) continue;
                    bool zface = (z == c[2] - r || z == c[2] + r);
                    for (i64 y = c[1] - r; y <= c[1] + r; ++y) {
                        if (y < 0 || y >= g.dims[1]) continue;
                        bool yface = zface || (y == c[1] - r || y == c[1] + r);
                        for (i64 xx = c[0] - r; xx <= c[0] + r; ++xx) {
                            if (xx < 0 || xx >= g.dims[0]) continue;
                            if (!yface && xx != c[0] - r && xx != c[0] + r) continue;
                            i64 cell = (z * g.dims[1] + y) * g.dims[0] + xx;
                            for (i64 t = g.start[cell]; t < g.start[cell + 1]; ++t) {
                                i32 j = g.items[t];
                                best.offer(dist2(x, pts + 3 * (i64)j), j);
                            }
                        }
                    }
                }
                if (best.full()) {
                    // distance from x to the faces of the visited block
                    double dmin = std::numeric_limits<double>::infinity();
                    bool all = true;
                    for (int a = 0; a < 3; ++a) {
                        double lo_face = g.lo[a] + (double)(c[a] - r) * g.cell;
                        double hi_face = g.lo[a] + (double)(c[a] + r + 1) * g.cell;
                        if (c[a] - r > 0) { dmin = std::min(dmin, x[a] - lo_face); all = false; }
                        if (c[a] + r + 1 < g.dims[a]) { dmin = std::min(dmin, hi_face - x[a]); all = false; }
                    }
                    if (all) break;
                    if (dmin > 0) {
                        double b2 = dmin * dmin * (1.0 - 1e-9);
                        if (best.d[k - 1] < b2) break;
                    }
                }
            }
            for (int t = 0; t < k; ++t) out[(size_t)q * k + t] = t < best.count ? best.j[t] : -1;
        }
    });
}

i64 nearest_other(const double* pts, i64 n, std::vector<double>& nn2, int nthreads) {
    std::vector<i32> nb;
    knn_grid(pts, n, pts, n, 3, nb, nthreads);
    nn2.resize(n);
    i64 dup = -1;
    for (i64 i = 0; i < n; ++i) {
        i32 j = nb[3 * i] == (i32)i ? nb[3 * i + 1] : nb[3 * i];
        nn2[i] = dist2(pts + 3 * i, pts + 3 * (i64)j);
        if (nn2[i] == 0.0 && dup < 0) dup = i;
    }
    return dup;
}

// ---------------------------------------------------------------------------------------
// O8: weighted sample elimination (Yuksel 2015), fixed-point weights.
// ---------------------------------------------------------------------------------------
// One elimination pass with weight radius R; false if it would have to eliminate a point of
// zero weight (no live neighbour within R: index ties would then decide and wipe out the
// lowest-index region), in which case the caller enlarges R.
// Neighbours within R on a hashed grid of cells of side >= 2R (only occupied cells stored):
// points sorted by cell key (LSD radix), cell key -> run of points by open addressing.  The
// neighbour set {j != i : d(i, j) < R} does not depend on the grid, and the weights are
// integers, so neither does anything below.
struct CellHash {
    double lo[3], cell;
    i64 dims[3];
    std::vector<uint64_t> key;  // sorted occupied cell keys
    std::vector<i64> start;     // run of cell q: items[start[q] .. start[q+1])
    std::vector<i32> items;
    std::vector<i64> slot;      // open addressing: index into key, -1 empty
    uint64_t mask;
    static uint64_t mix(uint64_t k) {
        k ^= k >> 33; k *= 0xff51afd7ed558ccdull; k ^= k >> 33; k *= 0xc4ceb9fe1a85ec53ull; k ^= k >> 33;
        return k;
    }
    void coords(const double* x, i64* c) const {
        for (int a = 0; a < 3; ++a) {
            i64 v = (i64)std::floor((x[a] - lo[a]) / cell);
            c[a] = std::min<i64>(std::max<i64>(v, 0), dims[a] - 1);
        }
    }
    void build(const double* p, i64 n, double R) {
        double hi[3];
        for (int a = 0; a < 3; ++a) lo[a] = hi[a] = p[a];
        for (i64 i = 0; i < n; ++i)
            for (int a = 0; a < 3; ++a) {
                lo[a] = std::min(lo[a], p[3 * i + a]);
                hi[a] = std::max(hi[a], p[3 * i + a]);
            }
        cell = R > 0 ? 2.0 * R * (1.0 + 1e-6) : 1.0;
        for (;;) {  // cells only grow (any side >= R is correct); keep keys below 2^60
            double tot = 1.0;
            for (int a = 0; a < 3; ++a) tot *= std::floor((hi[a] - lo[a]) / cell) + 1.0;
            if (tot < 1e18) break;
            cell *= 2.0;
        }
        for (int a = 0; a < 3; ++a) dims[a] = (i64)std::floor((hi[a] - lo[a]) / cell) + 1;
        std::vector<uint64_t> k0(n), k1(n);
        std::vector<i32> i0(n), i1(n);
        uint64_t kmax = 0;
        for (i64 i = 0; i < n; ++i) {
            i64 c[3];
            coords(p + 3 * i, c);
            k0[i] = (uint64_t)((c[2] * dims[1] + c[1]) * dims[0] + c[0]);
            i0[i] = (i32)i;
            kmax = std::max(kmax, k0[i]);
        }
        for (int sh = 0; sh < 64 && (kmax >> sh) != 0; sh += 16) {  // stable LSD radix, 16-bit digits
            std::vector<i64> cnt(65537, 0);
            for (i64 i = 0; i < n; ++i) cnt[((k0[i] >> sh) & 0xffff) + 1]++;
            for (int d = 0; d < 65536; ++d) cnt[d + 1] += cnt[d];
            for (i64 i = 0; i < n; ++i) {
                const i64 o = cnt[(k0[i] >> sh) & 0xffff]++;
                k1[o] = k0[i];
                i1[o] = i0[i];
            }
            k0.swap(k1);
            i0.swap(i1);
        }
        items = std::move(i0);
        key.clear();
        start.clear();
        for (i64 i = 0; i < n; ++i)
            if (i == 0 || k0[i] != k0[i - 1]) {
                key.push_back(k0[i]);
                start.push_back(i);
            }
        start.push_back(n);
        uint64_t cap = 16;
        while (cap < 2 * key.size()) cap <<= 1;
        mask = cap - 1;
        slot.assign(cap, -1);
        for (size_t q = 0; q < key.size(); ++q) {
            uint64_t h = mix(key[q]) & mask;
            while (slot[h] >= 0) h = (h + 1) & mask;
            slot[h] = (i64)q;
        }
    }
    i64 find(uint64_t k) const {  // index into key, or -1
        for (uint64_t h = mix(k) & mask;; h = (h + 1) & mask) {
            const i64 q = slot[h];
            if (q < 0) return -1;
            if (key[q] == k) return q;
        }
    }
    template <class F>
    void near(const double* x, F&& f) const {
        // cell side >= 2R (1 + 1e-6): the ball of radius R around x lies in x's cell and, per
        // axis, the neighbour on the side of the nearer face -- a 2 x 2 x 2 block
        i64 c[3], o[3];
        coords(x, c);
        for (int a = 0; a < 3; ++a) {
            const double f = (x[a] - lo[a]) - (double)c[a] * cell;
            o[a] = f < 0.5 * cell ? c[a] - 1 : c[a] + 1;
        }
        for (int m = 0; m < 8; ++m) {
            const i64 zz = (m & 4) ? o[2] : c[2], yy = (m & 2) ? o[1] : c[1], xx = (m & 1) ? o[0] : c[0];
            if (zz < 0 || zz >= dims[2] || yy < 0 || yy >= dims[1] || xx < 0 || xx >= dims[0]) continue;
            const i64 q = find((uint64_t)((zz * dims[1] + yy) * dims[0] + xx));
            if (q < 0) continue;
            for (i64 t = start[q]; t < start[q + 1]; ++t) f(items[t]);
        }
    }
};

// One elimination pass with weight radius R; false if it would have to eliminate a point of
// zero weight (no live neighbour within R: index ties would then decide and wipe out the
// lowest-index region), in which case the caller enlarges R.
static bool wse_pass(const double* pts, i64 n, i64 nt, double R, std::vector<i64>& keep, int nthreads) {
    keep.clear();
    CellHash g;
    g.build(pts, n, R);
    using wse_w = i64;  // O8: fixed-point weights, 2^40 per unit
    // neighbour CSR: per-thread lists over contiguous point ranges, then concatenated
    const int T = n >= 4096 ? std::max(1, nthreads) : 1;
    const double R2far = R * R * (1.0 + 1e-6);
    std::vector<std::vector<i32>> nj(T);
    std::vector<std::vector<wse_w>> nw(T);
    std::vector<i64> ptr(n + 1, 0);
    {
        std::vector<std::thread> th;
        for (int t = 0; t < T; ++t)
            th.emplace_back([&, t] {
                for (i64 i = n * t / T; i < n * (t + 1) / T; ++i) {
                    const size_t c0 = nj[t].size();
                    g.near(pts + 3 * i, [&](i32 j) {
                        if (j == (i32)i) return;
                        const double d2 = dist2(pts + 3 * i, pts + 3 * (i64)j);
                        if (d2 > R2far) return;  // sqrt(d2) > R for certain
                        double d = std::sqrt(d2);
                        if (!(d < R)) return;
                        double u = 1.0 - d / R;
                        double u2 = u * u;
                        double u4 = u2 * u2;
                        double u8 = u4 * u4;
                        nj[t].push_back(j);
                        nw[t].push_back((wse_w)std::floor(u8 * 1099511627776.0 + 0.5));  // 2^40
                    });
                    ptr[i + 1] = (i64)(nj[t].size() - c0);
                }
            });
        for (auto& x : th) x.join();
    }
    for (i64 i = 0; i < n; ++i) ptr[i + 1] += ptr[i];
    std::vector<i32> adj(ptr[n]);
    std::vector<wse_w> adjw(ptr[n]);
    {
        std::vector<std::thread> th;
        for (int t = 0; t < T; ++t)
            th.emplace_back([&, t] {
                const i64 o = ptr[n * t / T];
                std::copy(nj[t].begin(), nj[t].end(), adj.begin() + o);
                std::copy(nw[t].begin(), nw[t].end(), adjw.begin() + o);
            });
        for (auto& x : th) x.join();
    }
    std::vector<wse_w> weight(n, 0);
    for (i64 i = 0; i < n; ++i)
        for (i64 t = ptr[i]; t < ptr[i + 1]; ++t) weight[i] += adjw[t];

    // The elimination takes the live point of highest priority (weight desc, index asc) and
    // lowers its live neighbours' weights.  The popped priorities are strictly decreasing (the
    // top never rises: every other weight only falls), so the points eliminated are the
    // n - nt of highest priority at their pop, and a point whose priority beats every live
    // neighbour's pops with exactly that priority (no neighbour can pop before it).  So all
    // such local maxima are popped together, round after round (integer weights: the
    // neighbour updates commute), until no live point has positive weight; then the n - nt
    // highest pop priorities are selected.  The pass is degenerate (false) exactly when the
    // sequential loop would have met a zero-weight top: fewer than n - nt positive pops.
    const i64 ne = n - nt;
    std::vector<uint8_t> dead(n, 0);
    std::vector<i64> stamp(n, -1);  // round in which a point was last queued
    std::vector<i32> cand;
    cand.reserve(n);
    for (i64 i = 0; i < n; ++i)
        if (weight[i] > 0) cand.push_back((i32)i);
    struct Pop { wse_w w; i32 v; };
    std::vector<Pop> pops;
    pops.reserve(n);
    const int NT = std::max(1, nthreads);
    auto run = [&](i64 m, auto&& f) {  // f(t, b, e) over [0, m)
        const int k = m >= 16384 ? NT : 1;
        if (k == 1) { f(0, (i64)0, m); return; }
        std::vector<std::thread> th;
        for (int t = 0; t < k; ++t) th.emplace_back([&, t] { f(t, m * t / k, m * (t + 1) / k); });
        for (auto& x : th) x.join();
    };
    std::vector<std::vector<i32>> tl(NT);
    for (i64 round = 0; !cand.empty(); ++round) {
        // 1. local maxima among the candidates (read-only)
        for (auto& v : tl) v.clear();
        run((i64)cand.size(), [&](int t, i64 b, i64 e) {
            for (i64 q = b; q < e; ++q) {
                const i32 x = cand[q];
                const wse_w wx = weight[x];
                if (dead[x] || wx <= 0) continue;
                bool top = true;
                for (i64 r = ptr[x]; r < ptr[x + 1] && top; ++r) {
                    const i32 y = adj[r];
                    if (!dead[y] && (weight[y] > wx || (weight[y] == wx && y < x))) top = false;
                }
                if (top) tl[t].push_back(x);
            }
        });
        const size_t p0 = pops.size();
        for (auto& v : tl)
            for (i32 x : v) pops.push_back(Pop{weight[x], x});
        const i64 np_ = (i64)(pops.size() - p0);
        // 2. pop them, 3. lower their live neighbours' weights (exact integer updates)
        for (size_t q = p0; q < pops.size(); ++q) dead[pops[q].v] = 1;
        run(np_, [&](int, i64 b, i64 e) {
            for (i64 q = b; q < e; ++q) {
                const i32 x = pops[p0 + q].v;
                for (i64 r = ptr[x]; r < ptr[x + 1]; ++r)
                    if (!dead[adj[r]]) __atomic_fetch_sub(&weight[adj[r]], adjw[r], __ATOMIC_RELAXED);
            }
        });
        // 4. next candidates: live points within two hops of a popped point (only their
        //    neighbourhoods changed)
        for (auto& v : tl) v.clear();
        run(np_, [&](int t, i64 b, i64 e) {
            auto queue = [&](i32 y) {
                if (!dead[y] && __atomic_exchange_n(&stamp[y], round, __ATOMIC_RELAXED) != round) tl[t].push_back(y);
            };
            for (i64 q = b; q < e; ++q) {
                const i32 x = pops[p0 + q].v;
                for (i64 r = ptr[x]; r < ptr[x + 1]; ++r) {
                    const i32 y = adj[r];
                    if (dead[y]) continue;
                    queue(y);
                    for (i64 r2 = ptr[y]; r2 < ptr[y + 1]; ++r2) queue(adj[r2]);
                }
            }
        });
        cand.clear();
        for (auto& v : tl) cand.insert(cand.end(), v.begin(), v.end());
    }
    if ((i64)pops.size() < ne) return false;  // degenerate: R too small for this cloud (O8)
    std::nth_element(pops.begin(), pops.begin() + (ne - 1), pops.end(), [](const Pop& x, const Pop& y) {
        return x.w > y.w || (x.w == y.w && x.v < y.v);
    });
    std::fill(dead.begin(), dead.end(), 0);
    for (i64 q = 0; q < ne; ++q) dead[pops[q].v] = 1;
    keep.reserve(nt);
    for (i64 i = 0; i < n; ++i)
        if (!dead[i]) keep.push_back(i);
    return true;
}

// O8: R = 2 r_max with r_max = r_h sqrt(N / N_t), r_h = half the median nearest-other distance
double wse_initial_radius(const std::vector<double>& nn2, i64 n, i64 nt) {
    std::vector<double> s(n);
    for (i64 i = 0; i < n; ++i) s[i] = std::sqrt(nn2[i]);
    std::nth_element(s.begin(), s.begin() + (n - 1) / 2, s.end());
    double rh = 0.5 * s[(n - 1) / 2];
    double rmax = rh * std::sqrt((double)n / (double)nt);
    return 2.0 * rmax;
}

void wse_eliminate(const double* pts, i64 n, i64 nt, const std::vector<double>& nn2,
                   std::vector<i64>& keep, int nthreads) {
    keep.clear();
    if (nt >= n) {
        for (i64 i = 0; i < n; ++i) keep.push_back(i);
        return;
    }
    // O8: a degenerate pass (zero-weight elimination) restarts with R *= 1.25
    double R = wse_initial_radius(nn2, n, nt);
    for (int attempt = 0; attempt < 16; ++attempt, R *= 1.25)
        if (wse_pass(pts, n, nt, R, keep, nthreads)) return;
}

// ---------------------------------------------------------------------------------------
// ---------------------------------------------------------------------------------------
// Partition tables of one level for every rank (mgm_internal.h PartTables).
// ---------------------------------------------------------------------------------------
void partition_level(const HostCSR& L, const std::vector<int>& owner, const std::vector<i32>& colour, int ncol,
                     const HostCSR* Pj, const std::vector<int>* owner_c, const HostCSR* Pf,
                     const std::vector<int>* owner_f, int nranks, std::vector<PartTables>& out) {
    const i64 n = L.nrows;
    std::vector<std::vector<i64>> need(nranks);  // non-owned rows each rank reads
    for (i64 r = 0; r < n; ++r) {
        const int q = owner[r];
        for (i64 t = L.ptr[r]; t < L.ptr[r + 1]; ++t)
            if (owner[L.col[t]] != q) need[q].push_back(L.col[t]);
    }
    if (Pj && owner_c)  // R_j = P_j^T: coarse row c (owned by owner_c[c]) reads fine rows r with P_j[r][c] != 0
        for (i64 r = 0; r < n; ++r)
            for (i64 t = Pj->ptr[r]; t < Pj->ptr[r + 1]; ++t) {
                const int q = (*owner_c)[Pj->col[t]];
                if (owner[r] != q) need[q].push_back(r);
            }
    if (Pf && owner_f)  // P_{j-1}: fine row f (owned by owner_f[f]) reads this level's rows
        for (i64 f = 0; f < Pf->nrows; ++f) {
            const int q = (*owner_f)[f];
            for (i64 t = Pf->ptr[f]; t < Pf->ptr[f + 1]; ++t)
                if (owner[Pf->col[t]] != q) need[q].push_back(Pf->col[t]);
        }
    out.assign(nranks, PartTables());
    for (int q = 0; q < nranks; ++q) {
        auto& g = need[q];
        std::sort(g.begin(), g.end());
        g.erase(std::unique(g.begin(), g.end()), g.end());
        std::stable_sort(g.begin(), g.end(), [&](i64 a, i64 b) { return owner[a] < owner[b]; });
        out[q].ghosts = g;
    }
    for (i64 r = 0; r < n; ++r) out[owner[r]].rows.push_back(r);
    // send lists: rank q sends to p the rows of need[p] that q owns (need[p] is sorted by
    // (owner, row), so they are one contiguous run); colour slices by scanning colours
    for (int q = 0; q < nranks; ++q) {
        PartTables& T = out[q];
        T.send_off.assign(1, 0);
        T.recv_off.assign(1, 0);
        for (int p = 0; p < nranks; ++p) {
            if (p == q) continue;
            const auto& gp = out[p].ghosts;
            auto lo = std::lower_bound(gp.begin(), gp.end(), q, [&](i64 a, int v) { return owner[a] < v; });
            auto hi = std::upper_bound(gp.begin(), gp.end(), q, [&](int v, i64 a) { return v < owner[a]; });
            const auto& gq = T.ghosts;
            auto lo2 = std::lower_bound(gq.begin(), gq.end(), p, [&](i64 a, int v) { return owner[a] < v; });
            auto hi2 = std::upper_bound(gq.begin(), gq.end(), p, [&](int v, i64 a) { return v < owner[a]; });
            if (lo == hi && lo2 == hi2) continue;
            T.peers.push_back(p);
            const i64 s0 = (i64)T.send_rows.size();
            T.send_rows.insert(T.send_rows.end(), lo, hi);
            T.send_off.push_back((i64)T.send_rows.size());
            const i64 g0 = (i64)(lo2 - gq.begin()), g1 = (i64)(hi2 - gq.begin());
            T.recv_off.push_back(g1);
            // colour slices (rows ascending = colours ascending in lib order)
            auto slices = [&](const std::vector<i64>& v, i64 a, i64 b, std::vector<i64>& coff) {
                i64 k = a;
                for (int c = 0; c <= ncol; ++c) {
                    while (k < b && colour[v[(size_t)k]] < c) ++k;
                    coff.push_back(k);
                }
                coff.back() = b;
            };
            slices(T.send_rows, s0, (i64)T.send_rows.size(), T.send_coff);
            slices(gq, g0, g1, T.recv_coff);
            (void)g0;
        }
        // recv_off[0] must be the first peer's ghost start: ghosts are sorted by owner and every
        // owner != q in them is a peer, so the segments tile [0, nghost)
        if (!T.peers.empty()) T.recv_off[0] = 0;
    }
}

HostCSR transpose(const HostCSR& A) {
    HostCSR T;
    T.nrows = A.ncols;
    T.ncols = A.nrows;
    T.ptr.assign(T.nrows + 1, 0);
    for (i64 t = 0; t < A.nnz(); ++t) T.ptr[A.col[t] + 1]++;
    for (i64 r = 0; r < T.nrows; ++r) T.ptr[r + 1] += T.ptr[r];
    T.col.resize(A.nnz());
    T.val.resize(A.val.empty() ? 0 : A.nnz());
    std::vector<i64> fill(T.ptr.begin(), T.ptr.end() - 1);
    for (i64 i = 0; i < A.nrows; ++i)
        for (i64 t = A.ptr[i]; t < A.ptr[i + 1]; ++t) {
            i64 o = fill[A.col[t]]++;
            T.col[o] = (i32)i;
            if (!A.val.empty()) T.val[o] = A.val[t];
        }
    return T;
}

// O11: greedy colouring in index order on pattern(A) U pattern(A^T) minus the diagonal.
// O11: DSATUR colouring of sym(pattern(A)) minus the diagonal, then `passes`
// iterated-greedy passes (Culberson): each pass visits the vertices by descending colour of
// the previous pass (ties by index) and gives each the smallest colour unused by its
// neighbours already coloured in this pass, which never increases the colour count.
// (cfg3's hierarchy: ~15% fewer colours than greedy in Morton order, so fewer sequential
// GS steps per V-cycle, at equal MGM-GMRES iteration counts.)  passes < 0: greedy in Morton
// order only.
int colour_passes() {
    const char* e = std::getenv("MGM_COLOUR_PASSES");
    return e ? std::max(-1, std::atoi(e)) : 10;
}

// neighbours of each vertex in sym(pattern(A)) minus the diagonal: sorted, deduplicated.
// Pattern transpose, then each row's union sorted in its own slot (threads over rows) and
// compacted.
static int col_threads() { return std::max(1, std::min(64, (int)std::thread::hardware_concurrency())); }

static void sym_adjacency(const HostCSR& A, std::vector<i64>& np, std::vector<i32>& nb) {
    const i64 n = A.nrows, nnz = A.nnz();
    const int nt = col_threads();
    // pattern transpose on threads (atomic counters: the order inside a transposed row is
    // arbitrary, every row is sorted and deduplicated below)
    std::vector<i64> tp(n + 1, 0);
    parallel_for(n, nt, [&](i64 b, i64 e) {
        for (i64 t = A.ptr[b]; t < A.ptr[e]; ++t) __atomic_fetch_add(&tp[A.col[t] + 1], 1, __ATOMIC_RELAXED);
    });
    for (i64 r = 0; r < n; ++r) tp[r + 1] += tp[r];
    std::vector<i32> tc((size_t)nnz);
    {
        std::vector<i64> fill(tp.begin(), tp.end() - 1);
        parallel_for(n, nt, [&](i64 b, i64 e) {
            for (i64 i = b; i < e; ++i)
                for (i64 t = A.ptr[i]; t < A.ptr[i + 1]; ++t)
                    tc[(size_t)__atomic_fetch_add(&fill[A.col[t]], 1, __ATOMIC_RELAXED)] = (i32)i;
        });
    }
    std::vector<i32> tmp((size_t)(2 * nnz));
    std::vector<i64> cnt(n + 1, 0);
    parallel_for(n, nt, [&](i64 b, i64 e) {
        for (i64 i = b; i < e; ++i) {
            i32* o = tmp.data() + A.ptr[i] + tp[i];
            i32* q = o;
            for (i64 t = A.ptr[i]; t < A.ptr[i + 1]; ++t)
                if (A.col[t] != i) *q++ = A.col[t];
            for (i64 t = tp[i]; t < tp[i + 1]; ++t)
                if (tc[t] != i) *q++ = tc[t];
            std::sort(o, q);
            cnt[i + 1] = std::unique(o, q) - o;
        }
    });
    np.assign(n + 1, 0);
    for (i64 i = 0; i < n; ++i) np[i + 1] = np[i] + cnt[i + 1];
    nb.resize((size_t)np[n]);
    parallel_for(n, nt, [&](i64 b, i64 e) {
        for (i64 i = b; i < e; ++i)
            std::copy(tmp.data() + A.ptr[i] + tp[i], tmp.data() + A.ptr[i] + tp[i] + cnt[i + 1], nb.data() + np[i]);
    });
}

// The priority order (sat, deg, lower index) is total, so which vertex is taken next does not
// depend on the queue's layout.  It is packed into one 64-bit key per vertex,
// sat << 56 | deg << 31 | (2^31 - 1 - index) (larger key = higher priority; deg < 2^25,
// n < 2^31), so a comparison is one integer compare.  Vertices with sat = 0 sit in one array
// sorted by priority; a vertex whose sat becomes >= 1 (it then outranks every sat = 0 vertex)
// enters an indexed max-heap of keys, where later sat increments sift it up in place.
// next(): the heap's top while the heap is non-empty, else the array's next uncoloured
// sat = 0 vertex.  The heap holds only the colouring front, each vertex once.  W 64-bit words
// of used-colour mask per vertex: W = 1 first (a colour index reaching 64 returns -1 and the
// caller reruns with W = 4; the same choices either way).
template <int W>
static int dsatur_impl(i64 n, const std::vector<i64>& np, const std::vector<i32>& nb, std::vector<i32>& colour) {
    constexpr int CMAX = 64 * W;
    const uint64_t IMASK = 0x7fffffffull;
    // one record per vertex (the fields the neighbour loop touches share a cache line):
    // current key (sat in the top byte), used-colour mask, heap slot (-1: not in the heap),
    // colour (-1: uncoloured)
    struct alignas(W == 1 ? 32 : 64) VR {
        uint64_t key;
        uint64_t bits[W];
        i32 pos;
        i32 col;
    };
    std::vector<VR> vr((size_t)n);
    for (i64 v = 0; v < n; ++v) {
        VR& r = vr[(size_t)v];
        r.key = ((uint64_t)(np[v + 1] - np[v]) << 31) | (IMASK - (uint64_t)v);
        for (int q = 0; q < W; ++q) r.bits[q] = 0;
        r.pos = -1;
        r.col = -1;
    }
    std::vector<uint64_t> a((size_t)n);
    for (i64 i = 0; i < n; ++i) a[(size_t)i] = vr[(size_t)i].key;
    std::sort(a.begin(), a.end(), std::greater<uint64_t>());  // all sat = 0 here
    size_t ac = 0;
    std::vector<uint64_t> h;  // heap of keys
    auto vert = [&](uint64_t k) { return (i64)(IMASK - (k & IMASK)); };
    auto up = [&](i64 k, uint64_t key) {
        while (k > 0 && key > h[(k - 1) / 2]) {
            h[k] = h[(k - 1) / 2];
            vr[(size_t)vert(h[k])].pos = (i32)k;
            k = (k - 1) / 2;
        }
        h[k] = key;
        vr[(size_t)vert(key)].pos = (i32)k;
    };
    auto pop = [&]() {
        const uint64_t top = h[0], last = h.back();
        h.pop_back();
        vr[(size_t)vert(top)].pos = -1;
        if (h.empty()) return vert(top);
        const i64 m = (i64)h.size();
        i64 k = 0;
        for (;;) {
            const i64 l = 2 * k + 1, r = l + 1;
            i64 c = k;
            uint64_t best = last;
            if (l < m && h[l] > best) { c = l; best = h[l]; }
            if (r < m && h[r] > best) { c = r; best = h[r]; }
            if (c == k) break;
            h[k] = h[c];
            vr[(size_t)vert(h[k])].pos = (i32)k;
            k = c;
        }
        h[k] = last;
        vr[(size_t)vert(last)].pos = (i32)k;
        return vert(top);
    };
    int maxc = 0;
    for (i64 done = 0; done < n; ++done) {
        i64 v;
        if (!h.empty()) {
            v = pop();
        } else {
            for (;; ++ac) {
                const VR& r = vr[(size_t)vert(a[ac])];
                if (r.col < 0 && (r.key >> 56) == 0) break;
            }
            v = vert(a[ac++]);
        }
        VR& rv = vr[(size_t)v];
        int c = 0;
        while (c < CMAX && (rv.bits[c >> 6] >> (c & 63) & 1ull)) ++c;
        if (c >= CMAX) return -1;
        rv.col = c;
        maxc = std::max(maxc, c + 1);
        const uint64_t cb = 1ull << (c & 63);
        for (i64 t = np[v]; t < np[v + 1]; ++t) {
            VR& rw = vr[(size_t)nb[t]];
            uint64_t& word = rw.bits[c >> 6];
            if ((word & cb) || rw.col >= 0) continue;
            word |= cb;
            rw.key += 1ull << 56;  // sat + 1 (sat < 256: at most one per colour below CMAX)
            up(rw.pos < 0 ? (h.push_back(rw.key), (i64)h.size() - 1) : (i64)rw.pos, rw.key);
        }
    }
    colour.resize(n);
    for (i64 v = 0; v < n; ++v) colour[v] = vr[(size_t)v].col;
    return maxc;
}

// DSATUR (Brelaz): colour the uncoloured vertex of largest saturation (distinct colours among
// its neighbours in sym(pattern) minus the diagonal), ties by larger degree (distinct
// neighbours) then lower index, with the smallest colour unused by its neighbours.  Returns
// the colour count, or -1 if a colour index would reach 256 (the caller falls back).
static int dsatur_colouring(i64 n, const std::vector<i64>& np, const std::vector<i32>& nb, std::vector<i32>& colour) {
    if (n >= ((i64)1 << 31)) return -1;
    for (i64 v = 0; v < n; ++v)
        if (np[v + 1] - np[v] >= ((i64)1 << 25)) return -1;
    const int c = dsatur_impl<1>(n, np, nb, colour);
    return c > 0 ? c : dsatur_impl<4>(n, np, nb, colour);
}

// smallest colour not used by an already coloured neighbour of i (stamp: per-caller scratch)
static inline i32 first_free(i64 i, i64 q, const std::vector<i64>& np, const std::vector<i32>& nb,
                             const std::vector<i32>& colour, std::vector<i64>& stamp) {
    for (i64 t = np[i]; t < np[i + 1]; ++t) {
        const i32 c = colour[nb[t]];
        if (c < 0) continue;
        if ((size_t)c >= stamp.size()) stamp.resize(2 * c + 2, -1);
        stamp[c] = q;
    }
    i32 c = 0;
    while ((size_t)c < stamp.size() && stamp[c] == q) ++c;
    return c;
}

// Iterated-greedy passes visit the previous colour classes one after another; a class is an
// independent set of sym(pattern), so no vertex of a class sees another of the same class,
// and the class's vertices are coloured on threads with the result of the sequential visit.
int greedy_colouring(const HostCSR& A, std::vector<i32>& colour, int passes, int device) {
    const i64 n = A.nrows;
    std::vector<i64> np;
    std::vector<i32> nb;  // the symmetric adjacency, built once for every pass
    sym_adjacency(A, np, nb);
    int ncol = 0;
    // first colouring: DSATUR (or greedy in Morton order if DSATUR needs >= 256 colours;
    // passes < 0: plain greedy in Morton order only)
    const int pass0 = (passes >= 0 && (ncol = dsatur_colouring(n, np, nb, colour)) > 0) ? 1 : 0;
    if (pass0 == 0) {
        colour.assign(n, -1);
        std::vector<i64> stamp(256, -1);
        ncol = 0;
        for (i64 i = 0; i < n; ++i) {
            colour[i] = first_free(i, i, np, nb, colour, stamp);
            ncol = std::max(ncol, colour[i] + 1);
        }
    }
    const int nt = col_threads();
    if (device >= 0 && passes > 0 && ncol <= 255) {
        const char* e = std::getenv("MGM_IG_DEVICE_MIN");
        const i64 dmin = e ? std::atoll(e) : 65536;
        if (n >= dmin) {
            const int nc = ig_passes_device(n, np.data(), nb.data(), colour.data(), ncol, passes, device);
            if (nc > 0) return nc;
            std::fprintf(stderr, "[mgm] device colouring passes failed (%d); host passes\n", nc);
        }
    }
    std::vector<i64> order(n);
    for (int pass = 1; pass <= std::max(passes, 0); ++pass) {
        // descending previous colour, ascending index within a colour
        std::vector<i64> cnt(ncol + 1, 0);
        for (i64 i = 0; i < n; ++i) cnt[ncol - colour[i]]++;
        for (int c = 0; c < ncol; ++c) cnt[c + 1] += cnt[c];
        const std::vector<i64> cls(cnt.begin(), cnt.end());  // class k: order[cls[k] .. cls[k+1])
        for (i64 i = 0; i < n; ++i) order[cnt[ncol - 1 - colour[i]]++] = i;
        colour.assign(n, -1);
        int nc = 0;
        for (int k = 0; k < ncol; ++k) {
            const i64 b0 = cls[k], len = cls[k + 1] - cls[k];
            const int ntk = len >= 8192 ? nt : 1;
            std::vector<int> tmax(std::max(ntk, 1), 0);
            std::vector<std::thread> th;
            auto run = [&](int t) {
                std::vector<i64> stamp(256, -1);
                int m = 0;
                for (i64 q = b0 + len * t / ntk; q < b0 + len * (t + 1) / ntk; ++q) {
                    const i64 i = order[q];
                    colour[i] = first_free(i, q, np, nb, colour, stamp);
                    m = std::max(m, colour[i] + 1);
                }
                tmax[t] = m;
            };
            if (ntk > 1) {
                for (int t = 0; t < ntk; ++t) th.emplace_back(run, t);
                for (auto& x : th) x.join();
            } else {
                run(0);
            }
            for (int m : tmax) nc = std::max(nc, m);
        }
        ncol = nc;
    }
    return ncol;
}

static int lu_threads() {
    return std::max(1, std::min(64, (int)std::thread::hardware_concurrency()));
}

// Explicit inverse from the LU factors (column-major, pivots): column i solves P A x = e_i by
// forward (unit lower, ascending k) and backward substitution (x_r = (b_r - sum_{c > r,
// ascending} U_rc x_c) / U_rr), the same operations per column as the single-threaded loop it
// replaces; U is transposed to row-major first so the backward sums read contiguously, and
// the columns run on threads.  Ainv row-major.
void dense_inverse(const std::vector<double>& LU, const std::vector<i32>& piv, int m, std::vector<double>& Ainv,
                   int nthreads) {
    std::vector<double> U((size_t)m * m);  // row-major copy: U[r*m + c] = LU(r, c)
    for (int c = 0; c < m; ++c)
        for (int r = 0; r < m; ++r) U[(size_t)r * m + c] = LU[(size_t)c * m + r];
    Ainv.assign((size_t)m * m, 0.0);
    parallel_for(m, m >= 256 ? nthreads : 1, [&](i64 a, i64 b) {
        std::vector<double> bb(m);
        for (i64 i = a; i < b; ++i) {
            std::fill(bb.begin(), bb.end(), 0.0);
            bb[(size_t)i] = 1.0;
            for (int k = 0; k < m; ++k)
                if (piv[k] != k) std::swap(bb[k], bb[piv[k]]);
            for (int k = 0; k < m; ++k)
                for (int r = k + 1; r < m; ++r) bb[r] -= LU[(size_t)k * m + r] * bb[k];
            for (int r = m - 1; r >= 0; --r) {
                double acc = bb[r];
                const double* ur = U.data() + (size_t)r * m;
                for (int c = r + 1; c < m; ++c) acc -= ur[c] * bb[c];
                bb[r] = acc / ur[r];
            }
            for (int r = 0; r < m; ++r) Ainv[(size_t)r * m + i] = bb[r];
        }
    });
}

// Dense LU with partial pivoting (O13); ties -> lowest row.  Row-major in, column-major out.
i64 dense_lu_colmajor(std::vector<double>& A, int m, std::vector<double>& LU, std::vector<i32>& piv) {
    double amax = 0.0;
    for (double v : A) amax = std::max(amax, std::fabs(v));
    piv.resize(m);
    for (int k = 0; k < m; ++k) {
        int p = k;
        double pv = std::fabs(A[(i64)k * m + k]);
        for (int i = k + 1; i < m; ++i)
            if (std::fabs(A[(i64)i * m + k]) > pv) { pv = std::fabs(A[(i64)i * m + k]); p = i; }
        if (!(pv > 1e-14 * amax)) return k;
        piv[k] = p;
        if (p != k)
            for (int j = 0; j < m; ++j) std::swap(A[(i64)k * m + j], A[(i64)p * m + j]);
        double d = A[(i64)k * m + k];
        // rows below the pivot are independent: threads over rows (large coarsest levels)
        auto rows = [&](i64 a, i64 b) {
            for (i64 i = k + 1 + a; i < k + 1 + b; ++i) {
                double l = A[i * m + k] / d;
                A[i * m + k] = l;
                for (int j = k + 1; j < m; ++j) A[i * m + j] = A[i * m + j] - l * A[(i64)k * m + j];
            }
        };
        const i64 nr = m - k - 1;
        const int nt = (nr >= 256 && m >= 1024) ? std::min<i64>(lu_threads(), nr / 64) : 1;
        if (nt > 1) {
            std::vector<std::thread> th;
            for (int t = 0; t < nt; ++t) th.emplace_back([&, t] { rows(nr * t / nt, nr * (t + 1) / nt); });
            for (auto& x : th) x.join();
        } else {
            rows(0, nr);
        }
    }
    LU.resize((size_t)m * m);
    for (int i = 0; i < m; ++i)
        for (int j = 0; j < m; ++j) LU[(i64)j * m + i] = A[(i64)i * m + j];
    return -1;
}

}  // namespace mgm
