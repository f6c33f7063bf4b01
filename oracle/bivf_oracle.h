/*
 * TEST INFRASTRUCTURE — CPU restatement of the reference's online IVF-Flat
 * path, used ONLY as the checker by tests/, __graft_entry__.smoke() and the
 * cpu_baseline leg of bench.py.  Nothing in paper_2408_02937_b200/ links,
 * loads or calls it.
 *
 * Parity status:
 *   - l2 distance, quantizer, assign, insert (ids / duplicates / exhaustion),
 *     block layout, search + top-k, exceed, rearrangement, hops: PINNED against
 *     the reference itself (oracle/_ref, built from /root/reference/proj/src) and
 *     the committed fixtures in tests/golden/ (made by tests/golden/make_golden.py).
 *   - remove/delete and the inner-product metric: the reference has neither
 *      — "parity unpinned"; these rules ARE the spec
 *     (§Inner product).
 *
 * Every function cites the reference file:line it restates (paths under
 * /root/reference/proj).  Sequential, single-threaded, plain C11, compiled
 * with -ffp-contract=off so no FMA contraction changes the distance bits.
 */
#ifndef BIVF_ORACLE_H
#define BIVF_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_OK = 0, ORC_EINVAL = 1, ORC_EPOOL = 2, ORC_ECORRUPT = 3, ORC_ERANGE = 4 };
enum { ORC_L2 = 0, ORC_IP = 1 };

typedef struct orc_index orc_index;

/* distance.hpp:11-18 — ascending d, one fp32 accumulator, no FMA */
float orc_l2_sqr(const float* a, const float* b, uint32_t dim);
/* distance.hpp:22-30 — same over an interleaved slot, stride between dims */
float orc_l2_sqr_strided(const float* q, const float* base, uint32_t stride, uint32_t dim);
/* (extension) s = sum_d a_d*b_d ascending d, no FMA */
float orc_ip(const float* a, const float* b, uint32_t dim);
/* block_store.hpp:37-40 */
uint64_t orc_interleaved_offset(uint64_t slot, uint64_t d, uint64_t dim, uint64_t group);

orc_index* orc_create(uint32_t num_clusters, uint32_t dim, uint32_t block_capacity,
                      uint32_t num_blocks, uint32_t interleave_group,
                      uint64_t rearrange_threshold, int metric);
void orc_destroy(orc_index* h);
void orc_set_centroids(orc_index* h, const float* centroids);
/* ivf_index.cpp:61-82 build_offline; ids NULL -> ascending original index */
int orc_bulk_load(orc_index* h, const float* x, uint64_t n, const uint32_t* assignment,
                  const int64_t* ids);

uint32_t orc_assign(const orc_index* h, const float* y);           /* ivf_index.cpp:93-105 */
int orc_insert(orc_index* h, const float* x, uint64_t n, const int64_t* ids, int64_t* out_ids,
               uint64_t* inserted);                                  /* ivf_index.cpp:122-229 */
int orc_search(const orc_index* h, const float* q, uint64_t k, uint64_t nprobe,
               int64_t* out_ids, float* out_d, uint64_t* count);    /* ivf_index.cpp:262-298 */
int orc_probes(const orc_index* h, const float* q, uint64_t nprobe, uint32_t* out);
int orc_exceed(const orc_index* h, uint32_t c);                     /* ivf_index.cpp:300-311 */
int orc_rearrange(orc_index* h, uint32_t c);                        /* ivf_index.cpp:476-505 */
int orc_rearrange_sweep(orc_index* h);                              /* ivf_index.cpp:507-511 */
uint64_t orc_take_events(orc_index* h, uint64_t* out4, uint64_t cap);
int orc_remove(orc_index* h, const int64_t* ids, uint64_t n, uint64_t* removed,
               uint8_t* found);                                     /* extension */

/* introspection (ivf_index.hpp:84-103, block_store.hpp:75-132) */
uint64_t orc_size(const orc_index* h);
uint64_t orc_scalars_copied(const orc_index* h);
uint64_t orc_list_length(const orc_index* h, uint32_t c);
uint64_t orc_offline_count(const orc_index* h, uint32_t c);
uint64_t orc_hop_count(const orc_index* h, uint32_t c);
int32_t orc_online_head(const orc_index* h, uint32_t c);
uint32_t orc_online_blocks(const orc_index* h, uint32_t c);
uint64_t orc_allocated_blocks(const orc_index* h);
void orc_block_header(const orc_index* h, int32_t b, int32_t* out5);
void orc_block_ids(const orc_index* h, int32_t b, int64_t* out);
void orc_block_payload(const orc_index* h, int32_t b, float* out);
void orc_offline_segment(const orc_index* h, uint32_t c, int64_t* ids, float* payload);
uint64_t orc_cluster_contents(const orc_index* h, uint32_t c, int64_t* ids, float* vecs);
int64_t orc_next_id(const orc_index* h);

#ifdef __cplusplus
}
#endif
#endif
