/* TEST INFRASTRUCTURE ONLY — the CPU *checker* for the B200 back end.
 *
 * A plain-C restatement of the reference's SPDZ online-phase arithmetic
 * (/root/reference/proj/core, cited per function).  It is pinned against the
 * reference itself (oracle/_ref/libllspdz_ref.so, built from the unmodified
 * reference sources by oracle/Makefile) by tests/test_oracle_pin.py and against
 * the committed golden vectors in tests/golden/ by tests/test_oracle_golden.py.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library; the product (paper_2512_11112_b200) never does.
 *
 * Field: p = 2^32 - 5, elements u32 in [0, p).  All results are exact integer
 * arithmetic, so they are bit-identical to the reference by construction.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define P 4294967291ull
#define GAMMA 0x9e3779b97f4a7c15ull

/* ---- field.hpp:14-46 ---- */
static inline uint32_t fp_reduce(uint64_t v) { return (uint32_t)(v % P); }
static inline uint32_t fp_add(uint32_t a, uint32_t b) {
    uint64_t s = (uint64_t)a + b;
    if (s >= P) s -= P;
    return (uint32_t)s;
}
static inline uint32_t fp_sub(uint32_t a, uint32_t b) {
    return a >= b ? a - b : (uint32_t)((uint64_t)a + P - b);
}
static inline uint32_t fp_neg(uint32_t a) { return a == 0 ? 0 : (uint32_t)(P - a); }
static inline uint32_t fp_mul(uint32_t a, uint32_t b) { return (uint32_t)(((uint64_t)a * b) % P); }

uint32_t or_fp_add(uint32_t a, uint32_t b) { return fp_add(a, b); }
uint32_t or_fp_sub(uint32_t a, uint32_t b) { return fp_sub(a, b); }
uint32_t or_fp_mul(uint32_t a, uint32_t b) { return fp_mul(a, b); }
uint32_t or_fp_reduce(uint64_t v) { return fp_reduce(v); }

/* ---- hash.hpp:11-26 ---- */
static inline uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
uint64_t or_splitmix64(uint64_t* state) { return mix64(*state += GAMMA); }
uint64_t or_fnv1a64(const void* data, uint64_t len, uint64_t seed) {
    const uint8_t* p = (const uint8_t*)data;
    uint64_t h = seed;
    for (uint64_t i = 0; i < len; ++i) {
        h ^= p[i];
        h *= 1099511628211ull;
    }
    return h;
}

/* ---- std::mt19937_64 (the seeded input generator of tests/test_util.hpp:46-51) ---- */
typedef struct { uint64_t mt[312]; int idx; } mt64_t;
static void mt64_seed(mt64_t* s, uint64_t seed) {
    s->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        s->mt[i] = 6364136223846793005ull * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
    s->idx = 312;
}
static uint64_t mt64_next(mt64_t* s) {
    if (s->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            uint64_t x = (s->mt[i] & 0xFFFFFFFF80000000ull) | (s->mt[(i + 1) % 312] & 0x7FFFFFFFull);
            uint64_t xa = x >> 1;
            if (x & 1) xa ^= 0xB5026F5AA96619E9ull;
            s->mt[i] = s->mt[(i + 156) % 312] ^ xa;
        }
        s->idx = 0;
    }
    uint64_t y = s->mt[s->idx++];
    y ^= (y >> 29) & 0x5555555555555555ull;
    y ^= (y << 17) & 0x71D67FFFEDA60000ull;
    y ^= (y << 37) & 0xFFF7EEE000000000ull;
    y ^= y >> 43;
    return y;
}
void or_rand_field_vec(uint64_t n, uint64_t seed, uint32_t* out) {
    mt64_t* s = (mt64_t*)malloc(sizeof(mt64_t));
    mt64_seed(s, seed);
    for (uint64_t i = 0; i < n; ++i) out[i] = (uint32_t)(mt64_next(s) % P);
    free(s);
}

/* ---- Dealer (spdz.cpp:162-249): a stateful splitmix64 stream with rejection ---- */
typedef struct {
    int n;
    uint64_t prime;
    uint64_t rng;
    uint32_t alpha;
    uint32_t alpha_shares[64];
} or_dealer_t;

uint32_t or_dealer_random_element(or_dealer_t* d) { /* spdz.cpp:175-183 */
    const uint64_t bound = (~0ull / d->prime) * d->prime;
    uint64_t v;
    do {
        v = or_splitmix64(&d->rng);
    } while (v >= bound);
    return (uint32_t)(v % d->prime);
}

void or_dealer_init(or_dealer_t* d, int n, uint64_t seed, uint64_t prime) { /* spdz.cpp:162-173 */
    d->n = n;
    d->prime = prime;
    d->rng = seed;
    uint32_t sum = 0;
    for (int i = 1; i < n; ++i) {
        d->alpha_shares[i] = or_dealer_random_element(d);
        sum = (uint32_t)(((uint64_t)sum + d->alpha_shares[i]) % prime);
    }
    uint32_t key = or_dealer_random_element(d);
    d->alpha_shares[0] = (uint32_t)(((uint64_t)key + prime - sum) % prime);
    d->alpha = key;
}
uint64_t or_dealer_sizeof(void) { return sizeof(or_dealer_t); }
uint64_t or_dealer_rng_state(const or_dealer_t* d) { return d->rng; }

/* spdz.cpp:185-201; out_v/out_m party-major (n * len). */
void or_dealer_share(or_dealer_t* d, const uint32_t* xs, uint64_t len, uint32_t* out_v, uint32_t* out_m) {
    const uint64_t p = d->prime;
    for (uint64_t j = 0; j < len; ++j) {
        uint32_t vs = 0, ms = 0;
        for (int i = 1; i < d->n; ++i) {
            uint32_t v = or_dealer_random_element(d);
            uint32_t m = or_dealer_random_element(d);
            out_v[(uint64_t)i * len + j] = v;
            out_m[(uint64_t)i * len + j] = m;
            vs = (uint32_t)(((uint64_t)vs + v) % p);
            ms = (uint32_t)(((uint64_t)ms + m) % p);
        }
        uint32_t mac = (uint32_t)(((uint64_t)d->alpha * xs[j]) % p);
        out_v[j] = (uint32_t)(((uint64_t)xs[j] + p - vs) % p);
        out_m[j] = (uint32_t)(((uint64_t)mac + p - ms) % p);
    }
}

/* spdz.cpp:203-208 */
void or_dealer_share_random(or_dealer_t* d, uint64_t len, uint32_t* clear, uint32_t* out_v, uint32_t* out_m) {
    for (uint64_t j = 0; j < len; ++j) clear[j] = or_dealer_random_element(d);
    or_dealer_share(d, clear, len, out_v, out_m);
}

/* triple_store.cpp:248-287: make_dealer_stores draws each input mask as share_random(1);
   mv/mm party-major (n * count), clear[count]. */
void or_dealer_masks(or_dealer_t* d, uint64_t count, uint32_t* clear, uint32_t* mv, uint32_t* mm) {
    uint32_t v[64], m[64];
    for (uint64_t j = 0; j < count; ++j) {
        or_dealer_share_random(d, 1, clear + j, v, m);
        for (int i = 0; i < d->n; ++i) {
            mv[(uint64_t)i * count + j] = v[i];
            mm[(uint64_t)i * count + j] = m[i];
        }
    }
}

/* spdz.cpp:210-225; planes[6] each n*lanes (a.v a.m b.v b.m c.v c.m). */
void or_dealer_triples(or_dealer_t* d, uint64_t lanes, uint32_t* const* planes) {
    uint32_t* a = (uint32_t*)malloc(lanes * 4);
    uint32_t* b = (uint32_t*)malloc(lanes * 4);
    uint32_t* c = (uint32_t*)malloc(lanes * 4);
    for (uint64_t i = 0; i < lanes; ++i) {
        a[i] = or_dealer_random_element(d);
        b[i] = or_dealer_random_element(d);
        c[i] = (uint32_t)(((uint64_t)a[i] * b[i]) % d->prime);
    }
    or_dealer_share(d, a, lanes, planes[0], planes[1]);
    or_dealer_share(d, b, lanes, planes[2], planes[3]);
    or_dealer_share(d, c, lanes, planes[4], planes[5]);
    free(a);
    free(b);
    free(c);
}

/* spdz.cpp:227-249; planes: A.v A.m (n*rows*din) B.v B.m (n*din) C.v C.m (n*rows). */
void or_dealer_matrix_triples(or_dealer_t* d, uint32_t din, uint32_t rows, uint32_t* const* planes) {
    uint64_t cells = (uint64_t)din * rows;
    uint32_t* A = (uint32_t*)malloc(cells * 4);
    uint32_t* B = (uint32_t*)malloc((uint64_t)din * 4);
    uint32_t* Cc = (uint32_t*)malloc((uint64_t)rows * 4);
    for (uint64_t i = 0; i < cells; ++i) A[i] = or_dealer_random_element(d);
    for (uint32_t i = 0; i < din; ++i) B[i] = or_dealer_random_element(d);
    for (uint32_t r = 0; r < rows; ++r) {
        uint64_t acc = 0;
        for (uint32_t c = 0; c < din; ++c) {
            acc += ((uint64_t)A[(uint64_t)r * din + c] * B[c]) % d->prime;
            if (acc >= (1ull << 60)) acc %= d->prime;
        }
        Cc[r] = (uint32_t)(acc % d->prime);
    }
    or_dealer_share(d, A, cells, planes[0], planes[1]);
    or_dealer_share(d, B, din, planes[2], planes[3]);
    or_dealer_share(d, Cc, rows, planes[4], planes[5]);
    free(A);
    free(B);
    free(Cc);
}

/* ---- backend.cpp:25-84 / spdz.cpp:9-33 ---- */
void or_add_batch(const uint32_t* xv, const uint32_t* xm, const uint32_t* yv, const uint32_t* ym, uint64_t n,
                  int sub, uint32_t* zv, uint32_t* zm) {
    for (uint64_t i = 0; i < n; ++i) {
        zv[i] = sub ? fp_sub(xv[i], yv[i]) : fp_add(xv[i], yv[i]);
        zm[i] = sub ? fp_sub(xm[i], ym[i]) : fp_add(xm[i], ym[i]);
    }
}

/* backend.cpp:53-65 */
void or_mul_mask(const uint32_t* xv, const uint32_t* yv, const uint32_t* av, const uint32_t* bv, uint64_t n,
                 uint32_t* d, uint32_t* e) {
    for (uint64_t i = 0; i < n; ++i) {
        d[i] = fp_sub(xv[i], av[i]);
        e[i] = fp_sub(yv[i], bv[i]);
    }
}

/* spdz.cpp:77-96; tri: a.v a.m b.v b.m c.v c.m */
void or_beaver_combine(const uint32_t* const* t, const uint32_t* d, const uint32_t* e, uint64_t n, int party,
                       uint32_t alpha, uint32_t* zv, uint32_t* zm) {
    for (uint64_t i = 0; i < n; ++i) {
        uint32_t de = fp_mul(d[i], e[i]);
        uint32_t v = t[4][i];
        v = fp_add(v, fp_mul(d[i], t[2][i]));
        v = fp_add(v, fp_mul(e[i], t[0][i]));
        if (party == 0) v = fp_add(v, de);
        uint32_t m = t[5][i];
        m = fp_add(m, fp_mul(d[i], t[3][i]));
        m = fp_add(m, fp_mul(e[i], t[1][i]));
        m = fp_add(m, fp_mul(alpha, de));
        zv[i] = v;
        zm[i] = m;
    }
}

/* backend.cpp:76-84 */
void or_reduce_add(const uint32_t* xv, const uint32_t* xm, uint64_t n, uint32_t* zv, uint32_t* zm) {
    uint32_t v = 0, m = 0;
    for (uint64_t i = 0; i < n; ++i) {
        v = fp_add(v, xv[i]);
        m = fp_add(m, xm[i]);
    }
    *zv = v;
    *zm = m;
}

/* ---- public-constant rules, spdz.cpp:35-75 (+ runtime.cpp:36-39 scalar broadcast: klen==1) ----
 * op: 0 add_public 1 sub_public 2 rsub_public 3 mul_public 4 share_of_public (x ignored on input) */
void or_public_op(int op, uint32_t* xv, uint32_t* xm, uint64_t n, const uint32_t* k, uint64_t klen, int party,
                  uint32_t alpha) {
    for (uint64_t i = 0; i < n; ++i) {
        uint32_t ki = k[klen == 1 ? 0 : i];
        switch (op) {
            case 0:
                if (party == 0) xv[i] = fp_add(xv[i], ki);
                xm[i] = fp_add(xm[i], fp_mul(alpha, ki));
                break;
            case 1:
                if (party == 0) xv[i] = fp_sub(xv[i], ki);
                xm[i] = fp_sub(xm[i], fp_mul(alpha, ki));
                break;
            case 2:
                xv[i] = party == 0 ? fp_sub(ki, xv[i]) : fp_neg(xv[i]);
                xm[i] = fp_sub(fp_mul(alpha, ki), xm[i]);
                break;
            case 3:
                xv[i] = fp_mul(xv[i], ki);
                xm[i] = fp_mul(xm[i], ki);
                break;
            case 4:
                xv[i] = party == 0 ? ki : 0;
                xm[i] = fp_mul(alpha, ki);
                break;
        }
    }
}

/* ---- open: net.cpp:170-215 (absorb: acc = add(acc, reduce(peer))) ---- */
void or_open_sum(const uint32_t* own, const uint32_t* const* peers, int n_peers, uint64_t len, uint32_t* out) {
    for (uint64_t i = 0; i < len; ++i) {
        uint32_t acc = own[i];
        for (int p = 0; p < n_peers; ++p) acc = fp_add(acc, fp_reduce(peers[p][i]));
        out[i] = acc;
    }
}

/* ---- spdz.cpp:98-124 ---- mt: A.v A.m B.v B.m C.v C.m */
void or_matrix_combine(uint32_t din, uint32_t rows, const uint32_t* const* mt, const uint32_t* D,
                       const uint32_t* E, int party, uint32_t alpha, uint32_t* zv, uint32_t* zm) {
    for (uint32_t r = 0; r < rows; ++r) {
        uint64_t v = mt[4][r], m = mt[5][r], de = 0;
        const uint64_t base = (uint64_t)r * din;
        for (uint32_t c = 0; c < din; ++c) {
            v += fp_mul(D[base + c], mt[2][c]);
            v += fp_mul(mt[0][base + c], E[c]);
            m += fp_mul(D[base + c], mt[3][c]);
            m += fp_mul(mt[1][base + c], E[c]);
            de += fp_mul(D[base + c], E[c]);
            if (v >= (1ull << 60)) v %= P;
            if (m >= (1ull << 60)) m %= P;
            if (de >= (1ull << 60)) de %= P;
        }
        uint32_t der = (uint32_t)(de % P);
        uint32_t vr = (uint32_t)(v % P);
        if (party == 0) vr = fp_add(vr, der);
        zv[r] = vr;
        zm[r] = fp_add((uint32_t)(m % P), fp_mul(alpha, der));
    }
}

/* ---- secret x public linear, runtime.cpp:303-334 (before the bias exec_add) ----
 * w_public != 0: W public (wv only), x secret (xv,xm) -> y = W x on both planes.
 * w_public == 0: x public (xv only), W secret (wv,wm) -> y.v = W.v x, y.m = W.m x. */
void or_linear_one_public(uint32_t din, uint32_t dout, int w_public, const uint32_t* wv, const uint32_t* wm,
                          const uint32_t* xv, const uint32_t* xm, uint32_t* yv, uint32_t* ym) {
    for (uint32_t r = 0; r < dout; ++r) {
        uint64_t v = 0, m = 0;
        for (uint32_t c = 0; c < din; ++c) {
            uint64_t idx = (uint64_t)r * din + c;
            if (w_public) {
                v += fp_mul(wv[idx], xv[c]);
                m += fp_mul(wv[idx], xm[c]);
            } else {
                v += fp_mul(wv[idx], xv[c]);
                m += fp_mul(wm[idx], xv[c]);
            }
            if (v >= (1ull << 60)) v %= P;
            if (m >= (1ull << 60)) m %= P;
        }
        yv[r] = (uint32_t)(v % P);
        ym[r] = (uint32_t)(m % P);
    }
}

/* ---- linear.cpp:7-21 ---- returns tiles or -11 (SliceTooSmall) */
int64_t or_plan_tiles(uint32_t din, uint32_t dout, uint64_t slice, uint32_t* starts, uint32_t* counts) {
    if (din == 0 || dout == 0 || slice < din) return -11;
    uint32_t rpt = (uint32_t)(slice / din);
    if (rpt == 0) rpt = 1;
    int64_t k = 0;
    for (uint32_t r = 0; r < dout; r += rpt) {
        if (starts) starts[k] = r;
        if (counts) counts[k] = (dout - r < rpt) ? dout - r : rpt;
        ++k;
    }
    return k;
}

/* ---- MAC check, spdz.cpp:126-138 ----
 * Records sorted by (batch_id, lane); r_j = reduce(splitmix64 stream from coin). */
typedef struct { uint64_t batch; uint32_t lane, value, mac; } rec_t;
static int rec_cmp(const void* a, const void* b) {
    const rec_t* x = (const rec_t*)a;
    const rec_t* y = (const rec_t*)b;
    if (x->batch != y->batch) return x->batch < y->batch ? -1 : 1;
    return x->lane < y->lane ? -1 : (x->lane > y->lane ? 1 : 0);
}
uint32_t or_mac_sigma(uint64_t n, const uint64_t* batch, const uint32_t* lane, const uint32_t* value,
                      const uint32_t* mac, uint64_t coin, uint32_t alpha) {
    rec_t* r = (rec_t*)malloc((n ? n : 1) * sizeof(rec_t));
    for (uint64_t i = 0; i < n; ++i) r[i] = (rec_t){batch[i], lane[i], value[i], mac[i]};
    qsort(r, n, sizeof(rec_t), rec_cmp);  /* std::sort is unstable too; equal keys never occur in a log */
    uint64_t state = coin;
    uint32_t sigma = 0;
    for (uint64_t i = 0; i < n; ++i) {
        uint32_t rj = fp_reduce(or_splitmix64(&state));
        uint32_t diff = fp_sub(r[i].mac, fp_mul(alpha, r[i].value));
        sigma = fp_add(sigma, fp_mul(rj, diff));
    }
    free(r);
    return sigma;
}

/* Closed form of the same sum (verified there): the record of
 * global rank j (0-based, in (batch, lane) order) uses r_j = reduce(mix(coin +
 * (j+1)*GAMMA)).  Contiguous segment [j0, j0+len) with value/mac arrays. */
uint32_t or_mac_sigma_segment(uint64_t j0, uint64_t len, const uint32_t* value, const uint32_t* mac,
                              uint64_t coin, uint32_t alpha) {
    uint32_t sigma = 0;
    for (uint64_t i = 0; i < len; ++i) {
        uint32_t rj = fp_reduce(mix64(coin + (j0 + i + 1) * GAMMA));
        uint32_t diff = fp_sub(mac[i], fp_mul(alpha, value[i]));
        sigma = fp_add(sigma, fp_mul(rj, diff));
    }
    return sigma;
}

/* spdz.cpp:140-145 */
uint64_t or_commit_sigma(uint32_t sigma, uint64_t nonce) {
    uint8_t buf[12];
    for (int i = 0; i < 4; ++i) buf[i] = (uint8_t)(sigma >> (8 * i));
    for (int i = 0; i < 8; ++i) buf[4 + i] = (uint8_t)(nonce >> (8 * i));
    return or_fnv1a64(buf, 12, 1469598103934665603ull);
}

/* spdz.cpp:147-158: 0 ok, 10 MacCheckFailed */
int or_verify_sigmas(uint64_t n, const uint32_t* sig, const uint64_t* nonces, const uint64_t* commits) {
    uint32_t total = 0;
    for (uint64_t i = 0; i < n; ++i) {
        if (or_commit_sigma(sig[i], nonces[i]) != commits[i]) return 10;
        total = fp_add(total, sig[i]);
    }
    return total != 0 ? 10 : 0;
}

/* Beaver multiply of a full n-party lockstep simulation (spdz.cpp:77-96 with
 * the open of net.cpp:170-215), share planes party-major (n * L).  Used by the
 * host-logic tests to build share-level expectations. */
void or_sim_beaver(int n, uint64_t L, const uint32_t* xv, const uint32_t* xm, const uint32_t* yv,
                   const uint32_t* ym, const uint32_t* const* tri, const uint32_t* alphas, uint32_t* zv,
                   uint32_t* zm, uint32_t* d_open, uint32_t* e_open) {
    for (uint64_t i = 0; i < L; ++i) {
        uint32_t d = 0, e = 0;
        for (int p = 0; p < n; ++p) {
            uint64_t o = (uint64_t)p * L + i;
            d = fp_add(d, fp_sub(xv[o], tri[0][o]));
            e = fp_add(e, fp_sub(yv[o], tri[2][o]));
        }
        d_open[i] = d;
        e_open[i] = e;
    }
    for (int p = 0; p < n; ++p) {
        const uint32_t* tp[6];
        for (int k = 0; k < 6; ++k) tp[k] = tri[k] + (uint64_t)p * L;
        or_beaver_combine(tp, d_open, e_open, L, p, alphas[p], zv + (uint64_t)p * L, zm + (uint64_t)p * L);
    }
    (void)xm;
    (void)ym;
}

uint32_t or_dealer_alpha(const or_dealer_t* d) { return d->alpha; }
uint32_t or_dealer_alpha_share(const or_dealer_t* d, int i) { return d->alpha_shares[i]; }
