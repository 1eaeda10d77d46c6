/* oracle/tsg_oracle.c -- TEST INFRASTRUCTURE ONLY (never on the product path).
 *
 * Plain-C restatement of the tilemul reference's spGEMM path; see
 * tsg_oracle.h.  Pinned against the reference compiled in place
 * (oracle/_ref/libref_tilemul.so) and the reference's golden hash by
 * tests/test_oracle.py.  Build: make -C oracle (-ffp-contract=off, as the
 * reference's proj/CMakeLists.txt:12-14).
 */
#include "tsg_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------ binary16 */
/* half.cpp:12-36.  Decomposes the double directly (bit fields), rounds the
 * significand to the binary16 quantum of its binade (2^(e-10) for normals,
 * 2^-24 for subnormals) with ties to even, and keeps the sign of zero. */
double tsgo_round_to_half(double x, int* status) {
  *status = 0;
  if (!isfinite(x) || fabs(x) > 65504.0) {
    *status = 3;
    return 0.0;
  }
  if (x == 0.0) return x;
  uint64_t bits;
  memcpy(&bits, &x, 8);
  const int E = (int)((bits >> 52) & 0x7ff);
  if (E == 0) return copysign(0.0, x); /* |x| < 2^-1022: far below 2^-25 */
  const int e = E - 1023;
  const uint64_t sig = (1ull << 52) | (bits & ((1ull << 52) - 1));
  const int q = e >= -14 ? e - 10 : -24; /* quantum exponent */
  const int shift = 52 + q - e;           /* >= 42 */
  uint64_t f;
  if (shift >= 64) {
    f = 0; /* value < 2^-11 quanta: rounds to zero */
  } else {
    f = sig >> shift;
    const uint64_t rem = sig & ((1ull << shift) - 1);
    const uint64_t half = 1ull << (shift - 1);
    if (rem > half || (rem == half && (f & 1))) ++f;
  }
  if (f == 0) return copysign(0.0, x);
  const double r = ldexp((double)f, q);
  return x < 0 ? -r : r;
}

/* ------------------------------------------------------------ helpers */
typedef struct {
  int64_t rows, cols, nnz;
  int64_t* rp;
  int32_t* col;
  float* val;
} Csrf; /* binary16-valued fp32 CSR after rounding and zero dropping */

static int round_csr(int64_t m, int64_t n, const int64_t* rp, const int32_t* col,
                     const double* val, Csrf* out) {
  const int64_t nnz = m > 0 ? rp[m] : 0;
  out->rows = m;
  out->cols = n;
  out->rp = (int64_t*)malloc((size_t)(m + 1) * sizeof(int64_t));
  out->col = (int32_t*)malloc((size_t)(nnz ? nnz : 1) * sizeof(int32_t));
  out->val = (float*)malloc((size_t)(nnz ? nnz : 1) * sizeof(float));
  int64_t w = 0;
  out->rp[0] = 0;
  for (int64_t r = 0; r < m; ++r) {
    for (int64_t p = rp[r]; p < rp[r + 1]; ++p) {
      int st;
      const double h = tsgo_round_to_half(val[p], &st);
      if (st) return st;
      if (h == 0.0) continue; /* tile_format.cpp:87,98 / oracle.cpp:110-115 */
      out->col[w] = col[p];
      out->val[w] = (float)h;
      ++w;
    }
    out->rp[r + 1] = w;
  }
  out->nnz = w;
  return 0;
}

static void free_csr(Csrf* c) {
  free(c->rp);
  free(c->col);
  free(c->val);
}

static int cmp_i32(const void* a, const void* b) {
  const int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  return (x > y) - (x < y);
}

/* ------------------------------------------------------ mixed oracle */
/* oracle.cpp:33-70 (spgemm_rows) with the mixed accumulator of :102-121:
 * a dense sparse accumulator per output row; A's row is walked in column
 * order, so every output element receives its products in ascending k. */
int tsgo_spgemm_mixed(int64_t m, int64_t k, const int64_t* rpA, const int32_t* colA,
                      const double* valA, int64_t n, const int64_t* rpB, const int32_t* colB,
                      const double* valB, int64_t** rpC, int32_t** colC, float** valC,
                      int64_t* nnzC) {
  Csrf A, B;
  int st = round_csr(m, k, rpA, colA, valA, &A);
  if (st) {
    free_csr(&A);
    return st;
  }
  st = round_csr(k, n, rpB, colB, valB, &B);
  if (st) {
    free_csr(&A);
    free_csr(&B);
    return st;
  }
  float* acc = (float*)calloc((size_t)(n ? n : 1), sizeof(float));
  unsigned char* occ = (unsigned char*)calloc((size_t)(n ? n : 1), 1);
  int32_t* touched = (int32_t*)malloc((size_t)(n ? n : 1) * sizeof(int32_t));
  int64_t cap = 1024, w = 0;
  int64_t* rp = (int64_t*)malloc((size_t)(m + 1) * sizeof(int64_t));
  int32_t* col = (int32_t*)malloc((size_t)cap * sizeof(int32_t));
  float* val = (float*)malloc((size_t)cap * sizeof(float));
  rp[0] = 0;
  for (int64_t i = 0; i < m; ++i) {
    int64_t nt = 0;
    for (int64_t p = A.rp[i]; p < A.rp[i + 1]; ++p) {
      const int32_t kk = A.col[p];
      const float a = A.val[p];
      for (int64_t q = B.rp[kk]; q < B.rp[kk + 1]; ++q) {
        const int32_t j = B.col[q];
        if (!occ[j]) {
          occ[j] = 1;
          touched[nt++] = j;
        }
        const float prod = a * B.val[q]; /* exact: binary16 x binary16 */
        acc[j] = acc[j] + prod;          /* the only rounding; no FMA (-ffp-contract=off) */
      }
    }
    qsort(touched, (size_t)nt, sizeof(int32_t), cmp_i32);
    for (int64_t t = 0; t < nt; ++t) {
      const int32_t j = touched[t];
      if (acc[j] != 0.0f) {
        if (w == cap) {
          cap *= 2;
          col = (int32_t*)realloc(col, (size_t)cap * sizeof(int32_t));
          val = (float*)realloc(val, (size_t)cap * sizeof(float));
        }
        col[w] = j;
        val[w] = acc[j];
        ++w;
      }
      acc[j] = 0.0f;
      occ[j] = 0;
    }
    rp[i + 1] = w;
  }
  free(acc);
  free(occ);
  free(touched);
  free_csr(&A);
  free_csr(&B);
  *rpC = rp;
  *colC = col;
  *valC = val;
  *nnzC = w;
  return 0;
}

/* ------------------------------------------------------ tiles */
typedef struct {
  int64_t tile_rows, tile_cols, ntiles;
  int64_t* trp;      /* tile row pointer */
  int32_t* tcol;     /* tile column */
  uint16_t* rows;    /* T masks per tile: bit c of row r */
} Tiles;

typedef struct {
  int32_t tc;
  int16_t r, c;
} Ent;

static int cmp_ent(const void* a, const void* b) {
  const Ent* x = (const Ent*)a;
  const Ent* y = (const Ent*)b;
  if (x->tc != y->tc) return (x->tc > y->tc) - (x->tc < y->tc);
  if (x->r != y->r) return x->r - y->r;
  return x->c - y->c;
}

/* from_element_coo (tile_format.cpp:61-129) reduced to the structure:
 * tiles keyed (tile row, tile col), sorted, with their row masks. */
static void build_tiles(const Csrf* M, int T, Tiles* t) {
  t->tile_rows = (M->rows + T - 1) / T;
  t->tile_cols = (M->cols + T - 1) / T;
  t->trp = (int64_t*)calloc((size_t)(t->tile_rows + 1), sizeof(int64_t));
  int64_t cap = 1024;
  t->tcol = (int32_t*)malloc((size_t)cap * sizeof(int32_t));
  t->rows = (uint16_t*)malloc((size_t)cap * T * sizeof(uint16_t));
  t->ntiles = 0;
  for (int64_t I = 0; I < t->tile_rows; ++I) {
    const int64_t r0 = I * T, r1 = (r0 + T < M->rows) ? r0 + T : M->rows;
    const int64_t ne = M->rp[r1] - M->rp[r0];
    Ent* e = (Ent*)malloc((size_t)(ne ? ne : 1) * sizeof(Ent));
    int64_t w = 0;
    for (int64_t r = r0; r < r1; ++r)
      for (int64_t p = M->rp[r]; p < M->rp[r + 1]; ++p) {
        e[w].tc = M->col[p] / T;
        e[w].r = (int16_t)(r - r0);
        e[w].c = (int16_t)(M->col[p] % T);
        ++w;
      }
    qsort(e, (size_t)w, sizeof(Ent), cmp_ent);
    for (int64_t i = 0; i < w;) {
      const int32_t tc = e[i].tc;
      if (t->ntiles == cap) {
        cap *= 2;
        t->tcol = (int32_t*)realloc(t->tcol, (size_t)cap * sizeof(int32_t));
        t->rows = (uint16_t*)realloc(t->rows, (size_t)cap * T * sizeof(uint16_t));
      }
      uint16_t* rm = t->rows + t->ntiles * T;
      memset(rm, 0, (size_t)T * sizeof(uint16_t));
      for (; i < w && e[i].tc == tc; ++i) rm[e[i].r] |= (uint16_t)(1u << e[i].c);
      t->tcol[t->ntiles++] = tc;
    }
    t->trp[I + 1] = t->ntiles;
    free(e);
  }
}

static void free_tiles(Tiles* t) {
  free(t->trp);
  free(t->tcol);
  free(t->rows);
}

static uint32_t col_occ(const uint16_t* rm, int T) { /* OR of rows: non-empty columns */
  uint32_t o = 0;
  for (int r = 0; r < T; ++r) o |= rm[r];
  return o;
}

static uint32_t row_occ(const uint16_t* rm, int T) { /* non-empty rows */
  uint32_t o = 0;
  for (int r = 0; r < T; ++r)
    if (rm[r]) o |= 1u << r;
  return o;
}

/* Count-only restatement of enumerate_pairs (pipeline.cpp:37-60),
 * filter_zero_products (:62-70, tile_product_nonzero :23-35),
 * sort_and_segment (:72-109) and counting_pass (kernels.cpp:79-103):
 * per A tile row, a sparse accumulator over output tile columns J holds the
 * OR of the boolean products (boolean_tile_mm, pipeline.cpp:11-21). */
int tsgo_tile_stats(int T, int64_t m, int64_t k, const int64_t* rpA, const int32_t* colA,
                    const double* valA, int64_t n, const int64_t* rpB, const int32_t* colB,
                    const double* valB, uint64_t* out) {
  if (T != 8 && T != 16) return 1;
  Csrf A, B;
  int st = round_csr(m, k, rpA, colA, valA, &A);
  if (!st) st = round_csr(k, n, rpB, colB, valB, &B);
  if (st) return st;
  Tiles tA, tB;
  build_tiles(&A, T, &tA);
  build_tiles(&B, T, &tB);
  const int64_t tcols = tB.tile_cols;
  uint16_t* spa = (uint16_t*)calloc((size_t)(tcols ? tcols : 1) * T, sizeof(uint16_t));
  unsigned char* seen = (unsigned char*)calloc((size_t)(tcols ? tcols : 1), 1);
  int64_t* touched = (int64_t*)malloc((size_t)(tcols ? tcols : 1) * sizeof(int64_t));
  uint64_t raw = 0, filt = 0, segs = 0, counted = 0;
  /* tile_product_nonzero's row occupancy of every B tile, once (the test
     itself is unchanged, pipeline.cpp:23-35) */
  uint32_t* bro = (uint32_t*)malloc((size_t)(tB.ntiles ? tB.ntiles : 1) * sizeof(uint32_t));
  for (int64_t b = 0; b < tB.ntiles; ++b) bro[b] = row_occ(tB.rows + b * T, T);
  for (int64_t I = 0; I < tA.tile_rows; ++I) {
    int64_t nt = 0;
    for (int64_t a = tA.trp[I]; a < tA.trp[I + 1]; ++a) {
      const int32_t kk = tA.tcol[a];
      const uint16_t* ar = tA.rows + a * T;
      const uint32_t aco = col_occ(ar, T);
      raw += (uint64_t)(tB.trp[kk + 1] - tB.trp[kk]);
      for (int64_t b = tB.trp[kk]; b < tB.trp[kk + 1]; ++b) {
        const uint16_t* br = tB.rows + b * T;
        if (!(aco & bro[b])) continue;
        ++filt;
        const int32_t J = tB.tcol[b];
        if (!seen[J]) {
          seen[J] = 1;
          touched[nt++] = J;
        }
        uint16_t* acc = spa + (int64_t)J * T;
        /* boolean_tile_mm (pipeline.cpp:11-21): row r of the product = OR of
           B's rows q over the set bits q of A's row r */
        for (int r = 0; r < T; ++r)
          for (uint32_t bits = ar[r]; bits; bits &= bits - 1) acc[r] |= br[__builtin_ctz(bits)];
      }
    }
    segs += (uint64_t)nt;
    for (int64_t t = 0; t < nt; ++t) {
      uint16_t* acc = spa + touched[t] * T;
      for (int r = 0; r < T; ++r) {
        counted += (uint64_t)__builtin_popcount(acc[r]);
        acc[r] = 0;
      }
      seen[touched[t]] = 0;
    }
  }
  out[0] = (uint64_t)tA.ntiles;
  out[1] = (uint64_t)tB.ntiles;
  out[2] = raw;
  out[3] = filt;
  out[4] = segs;
  out[5] = counted;
  free(bro);
  free(spa);
  free(seen);
  free(touched);
  free_tiles(&tA);
  free_tiles(&tB);
  free_csr(&A);
  free_csr(&B);
  return 0;
}

/* ------------------------------------------------------ golden hash */
typedef struct {
  uint64_t h;
} Fnv;

static void fnv_bytes(Fnv* f, const void* p, size_t n) { /* corpus.hpp:177-184 */
  const unsigned char* b = (const unsigned char*)p;
  for (size_t i = 0; i < n; ++i) {
    f->h ^= b[i];
    f->h *= 1099511628211ull;
  }
}

typedef struct {
  int32_t tc;
  int32_t bit;
  float v;
} Ent8;

static int cmp_ent8(const void* a, const void* b) {
  const Ent8* x = (const Ent8*)a;
  const Ent8* y = (const Ent8*)b;
  if (x->tc != y->tc) return (x->tc > y->tc) - (x->tc < y->tc);
  return (x->bit > y->bit) - (x->bit < y->bit);
}

/* serialize_tiled(from_element_coo(C, Fp32Stored)) (tiled_io.cpp:55-76,
 * tile_format.cpp:61-129) streamed through FNV-1a without materialising
 * the byte string: header, then the five arrays in order. */
uint64_t tsgo_fnv_tiled8(int64_t m, int64_t n, const int64_t* rp, const int32_t* col,
                         const float* val) {
  const int64_t trows = (m + 7) / 8;
  /* pass 1: tiles per tile row, in order */
  int64_t cap = 1024, nt = 0;
  uint32_t* trow = (uint32_t*)malloc((size_t)cap * 4);
  uint32_t* tcol = (uint32_t*)malloc((size_t)cap * 4);
  uint64_t* bm = (uint64_t*)malloc((size_t)cap * 8);
  uint64_t* ei = (uint64_t*)malloc((size_t)cap * 8);
  int64_t nnz = m > 0 ? rp[m] : 0;
  float* elems = (float*)malloc((size_t)(nnz ? nnz : 1) * sizeof(float));
  int64_t ne = 0;
  for (int64_t I = 0; I < trows; ++I) {
    const int64_t r0 = I * 8, r1 = r0 + 8 < m ? r0 + 8 : m;
    const int64_t cnt = rp[r1] - rp[r0];
    Ent8* e = (Ent8*)malloc((size_t)(cnt ? cnt : 1) * sizeof(Ent8));
    int64_t w = 0;
    for (int64_t r = r0; r < r1; ++r)
      for (int64_t p = rp[r]; p < rp[r + 1]; ++p) {
        if (val[p] == 0.0f) continue; /* zeros are not stored */
        e[w].tc = col[p] / 8;
        e[w].bit = (int32_t)(8 * (r - r0) + col[p] % 8);
        e[w].v = val[p];
        ++w;
      }
    qsort(e, (size_t)w, sizeof(Ent8), cmp_ent8);
    for (int64_t i = 0; i < w;) {
      if (nt == cap) {
        cap *= 2;
        trow = (uint32_t*)realloc(trow, (size_t)cap * 4);
        tcol = (uint32_t*)realloc(tcol, (size_t)cap * 4);
        bm = (uint64_t*)realloc(bm, (size_t)cap * 8);
        ei = (uint64_t*)realloc(ei, (size_t)cap * 8);
      }
      const int32_t tc = e[i].tc;
      trow[nt] = (uint32_t)I;
      tcol[nt] = (uint32_t)tc;
      ei[nt] = (uint64_t)ne;
      bm[nt] = 0;
      for (; i < w && e[i].tc == tc; ++i) {
        bm[nt] |= 1ull << e[i].bit;
        elems[ne++] = e[i].v;
      }
      ++nt;
    }
    free(e);
  }
  Fnv f = {1469598103934665603ull};
  const uint32_t version = 1;
  const uint8_t kind = 1; /* Fp32Stored */
  const uint64_t hdr[4] = {(uint64_t)m, (uint64_t)n, (uint64_t)nt, (uint64_t)ne};
  fnv_bytes(&f, "TSPZ", 4);
  fnv_bytes(&f, &version, 4);
  fnv_bytes(&f, &kind, 1);
  fnv_bytes(&f, hdr, sizeof hdr);
  fnv_bytes(&f, trow, (size_t)nt * 4);
  fnv_bytes(&f, tcol, (size_t)nt * 4);
  fnv_bytes(&f, bm, (size_t)nt * 8);
  fnv_bytes(&f, ei, (size_t)nt * 8);
  fnv_bytes(&f, elems, (size_t)ne * 4);
  free(trow);
  free(tcol);
  free(bm);
  free(ei);
  free(elems);
  return f.h;
}

uint64_t tsgo_cbar(int64_t m, int64_t k, const int64_t* rpA, const int32_t* colA,
                   const int64_t* rpB) {
  uint64_t* cc = (uint64_t*)calloc((size_t)(k ? k : 1), sizeof(uint64_t));
  const int64_t nnz = m > 0 ? rpA[m] : 0;
  for (int64_t p = 0; p < nnz; ++p) cc[colA[p]]++;
  uint64_t s = 0;
  for (int64_t i = 0; i < k; ++i) s += cc[i] * (uint64_t)(rpB[i + 1] - rpB[i]);
  free(cc);
  return s;
}

void tsgo_free(void* p) { free(p); }
