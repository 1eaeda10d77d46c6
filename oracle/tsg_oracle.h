/* oracle/tsg_oracle.h -- TEST INFRASTRUCTURE ONLY (never on the product path).
 *
 * Plain-C restatement of the tilemul reference's spGEMM path, used as the
 * CPU checker by tests/ and as the "port" CPU baseline by bench.py.  Each
 * function cites the reference code it follows.  It is pinned against the
 * reference itself (oracle/_ref, compiled in place) and against the
 * reference's golden FNV-1a hash (proj/tests/test_cli.cpp:149-169) by
 * tests/test_oracle.py.
 */
#ifndef TSG_ORACLE_H
#define TSG_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* round_to_half (proj/src/half.cpp:12-36): RNE to binary16 in one step from
 * the double; *status = 3 (OverflowError) when |x| > 65504 or non-finite. */
double tsgo_round_to_half(double x, int* status);

/* dense_spgemm_mixed_ordered (proj/src/oracle.cpp:102-121 over
 * spgemm_rows :33-70): inputs rounded to binary16 (zeros / underflow
 * dropped), each product exact in fp32, one fp32 add per product in
 * ascending k, exact zeros dropped.  Output CSR arrays are malloc'd
 * (tsgo_free).  Returns 0, 3 (overflow) or 4 (dimension). */
int tsgo_spgemm_mixed(int64_t m, int64_t k, const int64_t* rpA, const int32_t* colA,
                      const double* valA, int64_t n, const int64_t* rpB, const int32_t* colB,
                      const double* valB, int64_t** rpC, int32_t** colC, float** valC,
                      int64_t* nnzC);

/* Tile-level symbolic statistics of C = A.B at tile size T in {8, 16}
 * (count-only restatement of enumerate_pairs / filter_zero_products /
 * sort_and_segment, proj/src/pipeline.cpp:37-109, and counting_pass,
 * proj/src/kernels.cpp:79-103): out[0] tiles(A), out[1] tiles(B),
 * out[2] raw pairs, out[3] filtered pairs, out[4] segments (output tiles
 * allocated), out[5] counted elements (symbolic nnz(C)).  Values are rounded
 * to binary16 and dropped when zero, as from_element_coo(Fp16Stored) does. */
int tsgo_tile_stats(int T, int64_t m, int64_t k, const int64_t* rpA, const int32_t* colA,
                    const double* valA, int64_t n, const int64_t* rpB, const int32_t* colB,
                    const double* valB, uint64_t* out);

/* FNV-1a (proj/tests/support/corpus.hpp:177-184) of the .tspz
 * serialisation (proj/src/tiled_io.cpp:55-76) of from_element_coo(C,
 * Fp32Stored) at T = 8 (proj/src/tile_format.cpp:61-129). */
uint64_t tsgo_fnv_tiled8(int64_t m, int64_t n, const int64_t* rp, const int32_t* col,
                         const float* val);

/* sum_k nnzA(:,k) * nnzB(k,:)  (proj/src/analytics.cpp:51-65, A != B). */
uint64_t tsgo_cbar(int64_t m, int64_t k, const int64_t* rpA, const int32_t* colA,
                   const int64_t* rpB);

void tsgo_free(void* p);

#ifdef __cplusplus
}
#endif
#endif
