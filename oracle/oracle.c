/*
 * oracle.c -- plain, slow, obviously-correct CPU oracle (C99, no CUDA).
 *
 * TEST INFRASTRUCTURE.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / `--impl reference` leg may load this file's library.  It
 * shares nothing with the CUDA path in paper_2410_18129_b200/csrc.
 *
 * Every function computes the plain definition it is named after; the
 * citations say which passage of /root/reference/PAPER.md (P:Lnnn) defines the
 * result.  No blocking, fusion or reordering: schoolbook products, Knuth's
 * algorithm D, the extended Euclidean algorithm, left-to-right binary
 * square-and-multiply, Miller-Rabin.  "parity unpinned": none -- every
 * function is pinned by tests/test_oracle.py.
 */
#include "oracle.h"

#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ helpers */

static uint32_t* zalloc(size_t n) {
    uint32_t* p = (uint32_t*)calloc(n ? n : 1, sizeof(uint32_t));
    if (!p) abort();
    return p;
}

static int top_len(const uint32_t* a, int n) { /* number of significant limbs */
    while (n > 0 && a[n - 1] == 0) n--;
    return n;
}

static int bn_is_zero(const uint32_t* a, int n) { return top_len(a, n) == 0; }

/* compare a (na limbs) with b (nb limbs): -1, 0, 1 */
static int bn_cmp(const uint32_t* a, int na, const uint32_t* b, int nb) {
    na = top_len(a, na);
    nb = top_len(b, nb);
    if (na != nb) return na < nb ? -1 : 1;
    for (int i = na - 1; i >= 0; i--)
        if (a[i] != b[i]) return a[i] < b[i] ? -1 : 1;
    return 0;
}

/* r = a + b over n limbs, returns carry out (r may alias a or b) */
static uint32_t bn_add(uint32_t* r, const uint32_t* a, const uint32_t* b, int n) {
    uint64_t c = 0;
    for (int i = 0; i < n; i++) {
        uint64_t s = (uint64_t)a[i] + b[i] + c;
        r[i] = (uint32_t)s;
        c = s >> 32;
    }
    return (uint32_t)c;
}

/* r = a - b over n limbs, returns borrow out */
static uint32_t bn_sub(uint32_t* r, const uint32_t* a, const uint32_t* b, int n) {
    uint32_t br = 0;
    for (int i = 0; i < n; i++) {
        uint64_t d = (uint64_t)a[i] - b[i] - br;
        r[i] = (uint32_t)d;
        br = (uint32_t)((d >> 32) & 1);
    }
    return br;
}

/* ------------------------------------------------------- multiplication */

/* Schoolbook product: c = a*b, na+nb limbs.  Result of alg:8SBmul. */
void o_mul(const uint32_t* a, int na, const uint32_t* b, int nb, uint32_t* c) {
    uint32_t* t = zalloc((size_t)na + nb);
    for (int i = 0; i < na; i++) {
        uint64_t carry = 0;
        for (int j = 0; j < nb; j++) {
            uint64_t p = (uint64_t)a[i] * b[j] + t[i + j] + carry;
            t[i + j] = (uint32_t)p;
            carry = p >> 32;
        }
        t[i + nb] = (uint32_t)carry;
    }
    memcpy(c, t, sizeof(uint32_t) * ((size_t)na + nb));
    free(t);
}

/* Square: c = a*a, 2n limbs.  Result of alg:8SBsqu: the definition a^2 = a*a. */
void o_sqr(const uint32_t* a, int n, uint32_t* c) { o_mul(a, n, a, n, c); }

/* ------------------------------------------------------------- division */

/* Knuth, TAOCP vol. 2, 4.3.1, algorithm D.  q: na limbs, r: nb limbs. */
int o_divmod(const uint32_t* a, int na, const uint32_t* b, int nb, uint32_t* q, uint32_t* r) {
    int n = top_len(b, nb);
    if (n == 0) return -1;
    int m = top_len(a, na);
    uint32_t* qq = zalloc((size_t)na + 1);
    uint32_t* rr = zalloc((size_t)nb);
    if (m < n) { /* a < b */
        memcpy(rr, a, sizeof(uint32_t) * (size_t)m);
    } else if (n == 1) { /* short division */
        uint64_t rem = 0;
        for (int j = m - 1; j >= 0; j--) {
            uint64_t cur = (rem << 32) | a[j];
            qq[j] = (uint32_t)(cur / b[0]);
            rem = cur % b[0];
        }
        rr[0] = (uint32_t)rem;
    } else {
        /* D1: normalise so that the divisor's top bit is set */
        int s = __builtin_clz(b[n - 1]);
        uint32_t* vn = zalloc((size_t)n);
        uint32_t* un = zalloc((size_t)m + 1);
        for (int i = n - 1; i >= 0; i--) {
            uint64_t v = ((uint64_t)b[i] << s) | (i > 0 ? ((uint64_t)b[i - 1] << s) >> 32 : 0);
            vn[i] = (uint32_t)v;
        }
        un[m] = (uint32_t)(((uint64_t)a[m - 1] << s) >> 32);
        for (int i = m - 1; i >= 0; i--) {
            uint64_t v = ((uint64_t)a[i] << s) | (i > 0 ? ((uint64_t)a[i - 1] << s) >> 32 : 0);
            un[i] = (uint32_t)v;
        }
        const uint64_t B = 1ull << 32;
        for (int j = m - n; j >= 0; j--) {
            /* D3: estimate qhat from the top two limbs, correct it at most twice */
            uint64_t num = ((uint64_t)un[j + n] << 32) | un[j + n - 1];
            uint64_t qhat = num / vn[n - 1];
            uint64_t rhat = num % vn[n - 1];
            while (qhat >= B || qhat * vn[n - 2] > ((rhat << 32) | un[j + n - 2])) {
                qhat--;
                rhat += vn[n - 1];
                if (rhat >= B) break;
            }
            /* D4: multiply and subtract */
            int64_t k = 0, t;
            for (int i = 0; i < n; i++) {
                uint64_t p = qhat * vn[i];
                t = (int64_t)un[i + j] - k - (int64_t)(p & 0xFFFFFFFFull);
                un[i + j] = (uint32_t)t;
                k = (int64_t)(p >> 32) - (t >> 32);
            }
            t = (int64_t)un[j + n] - k;
            un[j + n] = (uint32_t)t;
            /* D5/D6: if negative, add back */
            qq[j] = (uint32_t)qhat;
            if (t < 0) {
                qq[j]--;
                uint64_t c = 0;
                for (int i = 0; i < n; i++) {
                    uint64_t s2 = (uint64_t)un[i + j] + vn[i] + c;
                    un[i + j] = (uint32_t)s2;
                    c = s2 >> 32;
                }
                un[j + n] = (uint32_t)((uint64_t)un[j + n] + c);
            }
        }
        /* D8: unnormalise the remainder */
        for (int i = 0; i < n; i++) {
            uint64_t v = ((uint64_t)un[i] >> s) | (s ? ((uint64_t)un[i + 1] << (32 - s)) & 0xFFFFFFFFull : 0);
            rr[i] = (uint32_t)v;
        }
        free(vn);
        free(un);
    }
    if (q) memcpy(q, qq, sizeof(uint32_t) * (size_t)na);
    if (r) memcpy(r, rr, sizeof(uint32_t) * (size_t)nb);
    free(qq);
    free(rr);
    return 0;
}

/* ---------------------------------------------------- modular inverse */

/* Extended Euclid on (m, a mod m), tracking the coefficient of a modulo m:
 * invariant t_i * a == r_i (mod m).  x = a^-1 mod m (nm limbs), -1 if gcd != 1. */
int o_inv_mod(const uint32_t* a, int na, const uint32_t* m, int nm, uint32_t* x) {
    int W = (na > nm ? na : nm) + 1;
    if (bn_is_zero(m, nm)) return -1;
    uint32_t *r0 = zalloc(W), *r1 = zalloc(W), *t0 = zalloc(W), *t1 = zalloc(W);
    uint32_t *qt = zalloc(W), *rem = zalloc(W), *prod = zalloc(2 * (size_t)W), *tmp = zalloc(W);
    uint32_t *mm = zalloc(W);
    memcpy(mm, m, sizeof(uint32_t) * (size_t)nm);
    memcpy(r0, m, sizeof(uint32_t) * (size_t)nm);
    uint32_t* aw = zalloc(W);
    memcpy(aw, a, sizeof(uint32_t) * (size_t)na);
    o_divmod(aw, W, mm, W, NULL, r1); /* r1 = a mod m */
    t1[0] = 1;                       /* t0 = 0, t1 = 1 */
    if (bn_cmp(mm, W, t1, W) == 0) t1[0] = 0; /* modulus 1 */
    while (!bn_is_zero(r1, W)) {
        o_divmod(r0, W, r1, W, qt, rem); /* q = r0 / r1 */
        memcpy(r0, r1, sizeof(uint32_t) * (size_t)W);
        memcpy(r1, rem, sizeof(uint32_t) * (size_t)W);
        o_mul(qt, W, t1, W, prod); /* q*t1 mod m */
        uint32_t* qtm = zalloc(2 * (size_t)W);
        o_divmod(prod, 2 * W, mm, W, NULL, qtm);
        if (bn_cmp(t0, W, qtm, W) >= 0) {
            bn_sub(tmp, t0, qtm, W);
        } else {
            bn_add(tmp, t0, mm, W);
            bn_sub(tmp, tmp, qtm, W);
        }
        free(qtm);
        memcpy(t0, t1, sizeof(uint32_t) * (size_t)W);
        memcpy(t1, tmp, sizeof(uint32_t) * (size_t)W);
    }
    uint32_t one[1] = {1};
    int ok = (bn_cmp(r0, W, one, 1) == 0);
    if (ok && x) memcpy(x, t0, sizeof(uint32_t) * (size_t)nm);
    free(r0); free(r1); free(t0); free(t1); free(qt); free(rem); free(prod); free(tmp); free(mm); free(aw);
    return ok ? 0 : -1;
}

/* Bezout: a*x - b*y = g = gcd(a,b), x in [0,b), y >= 0 (all n limbs). */
int o_egcd(const uint32_t* a, const uint32_t* b, int n, uint32_t* x, uint32_t* y, uint32_t* g) {
    int W = n + 1;
    if (bn_is_zero(b, n)) return -1;
    uint32_t *r0 = zalloc(W), *r1 = zalloc(W), *t0 = zalloc(W), *t1 = zalloc(W);
    uint32_t *qt = zalloc(W), *rem = zalloc(W), *prod = zalloc(2 * (size_t)W), *tmp = zalloc(W);
    uint32_t *bb = zalloc(W), *aw = zalloc(W);
    memcpy(bb, b, sizeof(uint32_t) * (size_t)n);
    memcpy(aw, a, sizeof(uint32_t) * (size_t)n);
    memcpy(r0, b, sizeof(uint32_t) * (size_t)n);
    o_divmod(aw, W, bb, W, NULL, r1);
    t1[0] = 1;
    while (!bn_is_zero(r1, W)) {
        o_divmod(r0, W, r1, W, qt, rem);
        memcpy(r0, r1, sizeof(uint32_t) * (size_t)W);
        memcpy(r1, rem, sizeof(uint32_t) * (size_t)W);
        o_mul(qt, W, t1, W, prod);
        uint32_t* qtm = zalloc(2 * (size_t)W);
        o_divmod(prod, 2 * W, bb, W, NULL, qtm);
        if (bn_cmp(t0, W, qtm, W) >= 0) {
            bn_sub(tmp, t0, qtm, W);
        } else {
            bn_add(tmp, t0, bb, W);
            bn_sub(tmp, tmp, qtm, W);
        }
        free(qtm);
        memcpy(t0, t1, sizeof(uint32_t) * (size_t)W);
        memcpy(t1, tmp, sizeof(uint32_t) * (size_t)W);
    }
    /* r0 = g, t0*a == g (mod b).  If b | a then t0 == 0 and g == b: use x = 1. */
    if (bn_is_zero(t0, W)) t0[0] = 1;
    /* y = (a*x - g)/b exactly */
    uint32_t* ax = zalloc(2 * (size_t)W);
    o_mul(aw, W, t0, W, ax);
    uint32_t* gw = zalloc(2 * (size_t)W);
    memcpy(gw, r0, sizeof(uint32_t) * (size_t)W);
    bn_sub(ax, ax, gw, 2 * W);
    uint32_t* yy = zalloc(2 * (size_t)W);
    uint32_t* rr = zalloc(W);
    o_divmod(ax, 2 * W, bb, W, yy, rr);
    int ok = bn_is_zero(rr, W);
    if (x) memcpy(x, t0, sizeof(uint32_t) * (size_t)n);
    if (y) memcpy(y, yy, sizeof(uint32_t) * (size_t)n);
    if (g) memcpy(g, r0, sizeof(uint32_t) * (size_t)n);
    free(r0); free(r1); free(t0); free(t1); free(qt); free(rem); free(prod); free(tmp);
    free(bb); free(aw); free(ax); free(gw); free(yy); free(rr);
    return ok ? 0 : -1;
}

/* ------------------------------------------------- Montgomery constants */

/* Nprime = (-N)^-1 mod R and R2 = R^2 mod N with R = 2^(32L) ("precomputed values"). */
int o_setup(const uint32_t* N, int L, uint32_t* Nprime, uint32_t* R2) {
    uint32_t* R = zalloc((size_t)L + 1);
    R[L] = 1;
    uint32_t* inv = zalloc((size_t)L + 1);
    if (o_inv_mod(N, L, R, L + 1, inv) != 0) { free(R); free(inv); return -1; }
    /* Nprime = R - inv (inv != 0 since N odd) */
    if (Nprime) {
        uint32_t* np = zalloc((size_t)L + 1);
        bn_sub(np, R, inv, L + 1);
        memcpy(Nprime, np, sizeof(uint32_t) * (size_t)L);
        free(np);
    }
    if (R2) {
        uint32_t* RR = zalloc(2 * (size_t)L + 1);
        RR[2 * L] = 1;
        o_divmod(RR, 2 * L + 1, N, L, NULL, R2);
        free(RR);
    }
    free(R);
    free(inv);
    return 0;
}

/* x <- x * 2^-1 mod N (N odd, x < N): x/2 if x even, (x+N)/2 otherwise. */
static void half_mod(uint32_t* x, const uint32_t* N, int L) {
    uint32_t top = 0;
    if (x[0] & 1) top = bn_add(x, x, N, L);
    for (int i = 0; i < L; i++) {
        uint32_t hi = (i + 1 < L) ? x[i + 1] : top;
        x[i] = (x[i] >> 1) | (hi << 31);
    }
}

/* c = T * R^-1 mod N, T of 2L limbs: (T mod N) halved 32L times (R^-1 = (2^-1)^(32L)). */
int o_redc(const uint32_t* T, const uint32_t* N, int L, uint32_t* c) {
    if (!(N[0] & 1)) return -1;
    uint32_t* x = zalloc((size_t)L);
    if (o_divmod(T, 2 * L, N, L, NULL, x) != 0) { free(x); return -1; }
    for (int k = 0; k < 32 * L; k++) half_mod(x, N, L);
    memcpy(c, x, sizeof(uint32_t) * (size_t)L);
    free(x);
    return 0;
}

/* c = a*b*R^-1 mod N. */
int o_montmul(const uint32_t* a, const uint32_t* b, const uint32_t* N, int L, uint32_t* c) {
    uint32_t* T = zalloc(2 * (size_t)L);
    o_mul(a, L, b, L, T);
    int rc = o_redc(T, N, L, c);
    free(T);
    return rc;
}

/* ---------------------------------------------------- exponentiation */

/* y = x*y mod N helper: y, x < N (L limbs) */
static void mulmod(uint32_t* y, const uint32_t* x, const uint32_t* N, int L, uint32_t* scratch2L) {
    o_mul(y, L, x, L, scratch2L);
    o_divmod(scratch2L, 2 * L, N, L, NULL, y);
}

/* out = base^e mod N by left-to-right binary square-and-multiply (P:L748 Ensure line). */
int o_modexp(const uint32_t* base, const uint32_t* e, int ebits, const uint32_t* N, int L, uint32_t* out) {
    if (bn_is_zero(N, L)) return -1;
    uint32_t* T = zalloc(2 * (size_t)L);
    uint32_t* a = zalloc((size_t)L);
    uint32_t* y = zalloc((size_t)L);
    uint32_t* bw = zalloc(2 * (size_t)L);
    memcpy(bw, base, sizeof(uint32_t) * (size_t)L);
    o_divmod(bw, 2 * L, N, L, NULL, a); /* a = base mod N */
    /* y = 1 mod N */
    uint32_t* one = zalloc(2 * (size_t)L);
    one[0] = 1;
    o_divmod(one, 2 * L, N, L, NULL, y);
    for (int bit = ebits - 1; bit >= 0; bit--) {
        mulmod(y, y, N, L, T);
        if ((e[bit >> 5] >> (bit & 31)) & 1) mulmod(y, a, N, L, T);
    }
    memcpy(out, y, sizeof(uint32_t) * (size_t)L);
    free(T); free(a); free(y); free(bw); free(one);
    return 0;
}

/* ------------------------------------------------------ primality */

static uint64_t splitmix64(uint64_t* s) {
    uint64_t z = (*s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

static const uint32_t small_primes[] = {
    3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37, 41, 43, 47, 53, 59, 61, 67, 71, 73, 79, 83, 89, 97,
    101, 103, 107, 109, 113, 127, 131, 137, 139, 149, 151, 157, 163, 167, 173, 179, 181, 191, 193,
    197, 199, 211, 223, 227, 229, 233, 239, 241, 251};

/* Miller-Rabin (trial division first).  1 = probable prime, 0 = composite. */
int o_is_probable_prime(const uint32_t* n, int L, int rounds, uint64_t seed) {
    int ln = top_len(n, L);
    if (ln == 0) return 0;
    if (ln == 1 && n[0] < 4) return n[0] >= 2;
    if (!(n[0] & 1)) return 0;
    for (size_t k = 0; k < sizeof(small_primes) / sizeof(small_primes[0]); k++) {
        uint32_t p = small_primes[k], r;
        uint32_t pv[1] = {p};
        if (ln == 1 && n[0] == p) return 1;
        o_divmod(n, L, pv, 1, NULL, &r);
        if (r == 0) return 0;
    }
    /* n - 1 = d * 2^s */
    uint32_t* nm1 = zalloc((size_t)L);
    uint32_t one[1] = {1};
    memcpy(nm1, n, sizeof(uint32_t) * (size_t)L);
    nm1[0] -= 1; /* n odd: no borrow */
    (void)one;
    uint32_t* d = zalloc((size_t)L);
    memcpy(d, nm1, sizeof(uint32_t) * (size_t)L);
    int s = 0;
    while (!(d[0] & 1)) {
        for (int i = 0; i < L; i++) d[i] = (d[i] >> 1) | ((i + 1 < L ? d[i + 1] : 0) << 31);
        s++;
    }
    uint32_t *a = zalloc((size_t)L), *x = zalloc((size_t)L), *T = zalloc(2 * (size_t)L);
    uint32_t* nm3 = zalloc((size_t)L);
    uint32_t three[1] = {3};
    uint32_t* threew = zalloc((size_t)L);
    threew[0] = three[0];
    bn_sub(nm3, n, threew, L);
    uint64_t st = seed;
    int prime = 1;
    for (int r = 0; r < rounds && prime; r++) {
        /* a uniform-ish in [2, n-2] */
        uint32_t* raw = zalloc((size_t)L);
        for (int i = 0; i < L; i++) raw[i] = (uint32_t)splitmix64(&st);
        o_divmod(raw, L, nm3, L, NULL, a);
        free(raw);
        uint32_t two[1] = {2};
        uint32_t* tw = zalloc((size_t)L);
        tw[0] = two[0];
        bn_add(a, a, tw, L);
        free(tw);
        o_modexp(a, d, 32 * L, n, L, x);
        uint32_t* onew = zalloc((size_t)L);
        onew[0] = 1;
        if (bn_cmp(x, L, onew, L) == 0 || bn_cmp(x, L, nm1, L) == 0) { free(onew); continue; }
        free(onew);
        int witness = 1;
        for (int k = 1; k < s; k++) {
            mulmod(x, x, n, L, T);
            if (bn_cmp(x, L, nm1, L) == 0) { witness = 0; break; }
        }
        if (witness) prime = 0;
    }
    free(nm1); free(d); free(a); free(x); free(T); free(nm3); free(threew);
    return prime;
}

int o_gen_prime(int bits, uint64_t seed, uint32_t* out) {
    if (bits < 3) return -1;
    int L = (bits + 31) / 32;
    uint64_t st = seed;
    uint32_t* c = zalloc((size_t)L);
    for (;;) {
        for (int i = 0; i < L; i++) c[i] = (uint32_t)splitmix64(&st);
        int tb = (bits - 1) & 31;
        c[L - 1] &= (tb == 31) ? 0xFFFFFFFFu : ((1u << (tb + 1)) - 1);
        c[L - 1] |= 1u << tb;
        c[0] |= 1;
        if (o_is_probable_prime(c, L, 40, splitmix64(&st))) break;
    }
    memcpy(out, c, sizeof(uint32_t) * (size_t)L);
    free(c);
    return 0;
}

/* ------------------------------------------- paper routes (readings) */

/* alg:montred, literally: q = T*N' mod R; C = (T + q*N) / R. */
int o_montred_classic(const uint32_t* T, const uint32_t* N, const uint32_t* Nprime, int L, uint32_t* C) {
    uint32_t* tn = zalloc(2 * (size_t)L);
    o_mul(T, L, Nprime, L, tn);                 /* T mod R times N' ... */
    uint32_t* q = zalloc((size_t)L);
    memcpy(q, tn, sizeof(uint32_t) * (size_t)L); /* ... mod R */
    uint32_t* qN = zalloc(2 * (size_t)L + 1);
    o_mul(q, L, N, L, qN);
    uint32_t* S = zalloc(2 * (size_t)L + 1);
    memcpy(S, T, sizeof(uint32_t) * 2 * (size_t)L);
    bn_add(S, S, qN, 2 * L + 1);
    int ok = bn_is_zero(S, L); /* exact division by R */
    memcpy(C, S + L, sizeof(uint32_t) * ((size_t)L + 1));
    free(tn); free(q); free(qN); free(S);
    return ok ? 0 : -1;
}

/* alg:trunc_montred with Theorem 2 read as SURVEY 8(c) A6/A7. */
int o_montred_truncated(const uint32_t* T, const uint32_t* N, const uint32_t* Nprime, int L,
                        uint32_t* C, uint32_t* qnhat_out) {
    /* line 1: q = T*N' mod R */
    uint32_t* tn = zalloc(2 * (size_t)L);
    o_mul(T, L, Nprime, L, tn);
    uint32_t* q = tn; /* low L limbs */
    /* line 2: qnhat = floor(q*N/R) from the partial products of weight >= L-1 (Theorem 2).
     * col[k] = sum_{i+j=k} lo(q_i N_j) + sum_{i+j=k-1} hi(q_i N_j), for k = L-1 .. 2L-1
     * (eq:qn for k = L-1, eq:qnhat for k >= L). */
    uint64_t* col = (uint64_t*)calloc(2 * (size_t)L + 1, sizeof(uint64_t));
    for (int i = 0; i < L; i++)
        for (int j = 0; j < L; j++) {
            uint64_t p = (uint64_t)q[i] * N[j];
            int k = i + j;
            if (k >= L - 1) col[k] += (uint32_t)p;
            if (k + 1 >= L - 1) col[k + 1] += p >> 32;
        }
    /* eq:TqN: word L-1 of T+qN is zero.  With b = [T mod 2^(32(L-1)) != 0] (A6), the word
     * L-1 of (qN mod R) is K = (-T[L-1] - b) mod 2^32, so the unknown carry Yc into column
     * L-1 satisfies (S + Yc) mod 2^32 = K, and the carry out of column L-1 is
     * floor(S/2^32) + [S mod 2^32 > K] (A7). */
    uint64_t S = col[L - 1];
    uint32_t b = !bn_is_zero(T, L - 1);
    uint32_t K = (uint32_t)(0u - T[L - 1] - b);
    uint64_t carry = (S >> 32) + (((uint32_t)S > K) ? 1 : 0);
    uint32_t* qnhat = zalloc((size_t)L + 1);
    for (int k = L; k <= 2 * L - 1; k++) {
        uint64_t v = col[k] + carry; /* col[k] < 2^39, carry < 2^39: no overflow */
        qnhat[k - L] = (uint32_t)v;
        carry = v >> 32;
    }
    qnhat[L] = (uint32_t)carry; /* zero since floor(qN/R) < N < R */
    /* line 3: c_add = OR of T[0..L-1]  (eq:c_add) */
    uint32_t c_add = !bn_is_zero(T, L);
    /* line 4: C = floor(T/R) + qnhat + c_add */
    uint32_t* Cw = zalloc((size_t)L + 1);
    memcpy(Cw, T + L, sizeof(uint32_t) * (size_t)L);
    bn_add(Cw, Cw, qnhat, L + 1);
    uint32_t* ca = zalloc((size_t)L + 1);
    ca[0] = c_add;
    bn_add(Cw, Cw, ca, L + 1);
    memcpy(C, Cw, sizeof(uint32_t) * ((size_t)L + 1));
    if (qnhat_out) memcpy(qnhat_out, qnhat, sizeof(uint32_t) * ((size_t)L + 1));
    free(tn); free(col); free(qnhat); free(Cw); free(ca);
    return 0;
}

/* alg:8BlockMontRed, the CIOS-inspired interleaved Montgomery multiplication,
 * step by step in 32-bit words (the paper's 52-bit word becomes a 32-bit limb; only
 * n0' = N' mod 2^32 is used):
 *   Y <- a[0]*B;  q <- Y mod 2^32 * n0' mod 2^32;  Y <- (Y + q*N) / 2^32     (lines 2-4)
 *   for i = 1 .. L-1:  Y <- Y + a[i]*B;  q <- ...;  Y <- (Y + q*N) / 2^32      (lines 5-9)
 * Y has L+2 limbs of room; the result (returned with L+1 limbs) is < 2N for a, b < N. */
int o_montmul_cios(const uint32_t* a, const uint32_t* B, const uint32_t* N, uint32_t n0p, int L, uint32_t* C) {
    const size_t W = (size_t)L + 2;
    uint32_t* Y = zalloc(W);
    uint32_t* t = zalloc(W);
    for (int i = 0; i < L; i++) {
        /* Y <- Y + a[i]*B */
        memset(t, 0, sizeof(uint32_t) * W);
        o_mul(&a[i], 1, B, L, t);
        bn_add(Y, Y, t, (int)W);
        /* q <- |Y|_{2^32} * n0' mod 2^32 */
        uint32_t q = Y[0] * n0p;
        /* Y <- (Y + q*N) / 2^32 : the low word becomes zero, then shift one word down */
        memset(t, 0, sizeof(uint32_t) * W);
        o_mul(&q, 1, N, L, t);
        bn_add(Y, Y, t, (int)W);
        if (Y[0] != 0) { free(Y); free(t); return -1; }
        memmove(Y, Y + 1, sizeof(uint32_t) * (W - 1));
        Y[W - 1] = 0;
    }
    memcpy(C, Y, sizeof(uint32_t) * ((size_t)L + 1));
    free(Y); free(t);
    return 0;
}

/* Batched CRT-RSA private-key operation (the paper's motivating use; SURVEY
 * 8(f) f4), step by step with plain definitions (Garner recombination):
 *   c_p = c mod p, c_q = c mod q;  m_p = c_p^dp mod p,  m_q = c_q^dq mod q;
 *   h = qinv*(m_p - m_q) mod p;  m = m_q + h*q   (= c^d mod pq for d = dp mod p-1, dq mod q-1).
 * c and m have 2*Lh limbs (c < p*q); p, q, dp, dq, qinv have Lh limbs; ebits = bits of dp, dq. */
int o_rsa_crt(const uint32_t* c, const uint32_t* p, const uint32_t* q, const uint32_t* dp, const uint32_t* dq,
              const uint32_t* qinv, int Lh, int ebits, uint32_t* m) {
    const size_t H = (size_t)Lh;
    uint32_t* cp = zalloc(H);
    uint32_t* cq = zalloc(H);
    uint32_t* mp = zalloc(H);
    uint32_t* mq = zalloc(H);
    uint32_t* w = zalloc(2 * H);
    uint32_t* t = zalloc(H + 1);
    uint32_t* d = zalloc(H + 1);
    uint32_t* h = zalloc(H);
    int rc = 0;
    rc |= o_divmod(c, 2 * Lh, p, Lh, NULL, cp);
    rc |= o_divmod(c, 2 * Lh, q, Lh, NULL, cq);
    rc |= o_modexp(cp, dp, ebits, p, Lh, mp);
    rc |= o_modexp(cq, dq, ebits, q, Lh, mq);
    /* t = m_q mod p */
    memcpy(w, mq, sizeof(uint32_t) * H);
    memset(w + H, 0, sizeof(uint32_t) * H);
    rc |= o_divmod(w, 2 * Lh, p, Lh, NULL, t);
    /* d = (m_p - t) mod p, in [0, p) */
    memcpy(d, mp, sizeof(uint32_t) * H);
    d[H] = 0;
    t[H] = 0;
    if (bn_cmp(d, Lh + 1, t, Lh + 1) < 0) {
        uint32_t* pw = zalloc(H + 1);
        memcpy(pw, p, sizeof(uint32_t) * H);
        bn_add(d, d, pw, Lh + 1);
        free(pw);
    }
    bn_sub(d, d, t, Lh + 1);
    /* h = qinv * d mod p */
    o_mul(qinv, Lh, d, Lh, w);
    rc |= o_divmod(w, 2 * Lh, p, Lh, NULL, h);
    /* m = m_q + h*q  (< p*q: no reduction) */
    o_mul(h, Lh, q, Lh, w);
    uint32_t* mq2 = zalloc(2 * H);
    memcpy(mq2, mq, sizeof(uint32_t) * H);
    bn_add(m, w, mq2, 2 * Lh);
    free(mq2); free(cp); free(cq); free(mp); free(mq); free(w); free(t); free(d); free(h);
    return rc ? -1 : 0;
}

/* ------------------------------------------------------ batch drivers */

typedef struct {
    int kind; /* 0 modexp, 1 montmul */
    const uint32_t *x, *y, *N;
    int ebits, L;
    uint32_t* out;
    size_t begin, end;
    int rc;
} job_t;

static void* worker(void* p) {
    job_t* j = (job_t*)p;
    size_t L = (size_t)j->L;
    size_t eL = (size_t)((j->ebits + 31) / 32);
    for (size_t k = j->begin; k < j->end; k++) {
        int rc;
        if (j->kind == 0)
            rc = o_modexp(j->x + k * L, j->y + k * eL, j->ebits, j->N + k * L, j->L, j->out + k * L);
        else
            rc = o_montmul(j->x + k * L, j->y + k * L, j->N + k * L, j->L, j->out + k * L);
        if (rc) j->rc = rc;
    }
    return NULL;
}

static int run_batch(int kind, const uint32_t* x, const uint32_t* y, int ebits, const uint32_t* N, int L,
                     uint32_t* out, size_t count, int threads) {
    if (threads < 1) threads = 1;
    if ((size_t)threads > count) threads = count ? (int)count : 1;
    pthread_t* th = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
    job_t* jobs = (job_t*)calloc((size_t)threads, sizeof(job_t));
    size_t per = (count + threads - 1) / threads;
    for (int t = 0; t < threads; t++) {
        jobs[t] = (job_t){kind, x, y, N, ebits, L, out, t * per, (t + 1) * per, 0};
        if (jobs[t].begin > count) jobs[t].begin = count;
        if (jobs[t].end > count) jobs[t].end = count;
        pthread_create(&th[t], NULL, worker, &jobs[t]);
    }
    int rc = 0;
    for (int t = 0; t < threads; t++) {
        pthread_join(th[t], NULL);
        if (jobs[t].rc) rc = jobs[t].rc;
    }
    free(th);
    free(jobs);
    return rc;
}

int o_batch_modexp(const uint32_t* base, const uint32_t* e, int ebits, const uint32_t* N, int L,
                   uint32_t* out, size_t count, int threads) {
    return run_batch(0, base, e, ebits, N, L, out, count, threads);
}

int o_batch_montmul(const uint32_t* a, const uint32_t* b, const uint32_t* N, int L,
                    uint32_t* c, size_t count, int threads) {
    return run_batch(1, a, b, 0, N, L, c, count, threads);
}
