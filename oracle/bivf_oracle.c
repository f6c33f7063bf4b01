/*
 * TEST INFRASTRUCTURE — CPU restatement of the reference's online IVF-Flat
 * path (see bivf_oracle.h for the scope and parity status).  It is the
 * checker for the CUDA product in paper_2408_02937_b200/, never part of it.
 *
 * State mirrors the reference's ClusterIndex (ivf_index.hpp:105-169) and
 * CentralMemoryPool (block_store.hpp:166-188): per-cluster offline segments
 * in the 32-way interleaved layout, a pre-split arena of blocks with
 * {prev,next,committed,owner,merged} headers, and per-cluster online lists
 * {length, head, tail, block count, fail flag}.
 */
#include "bivf_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    int64_t* keys;
    uint64_t cap, used;
} idset;

struct orc_index {
    uint32_t C, D, T, G, nblk_total, metric;
    uint64_t threshold;
    uint64_t groups_per_block, payload_scalars;
    float* centroids;
    /* offline segments */
    uint64_t* off_count;
    int64_t** off_ids;
    float** off_pay;
    /* pool */
    float* arena;
    int64_t* bids;
    int32_t *prev, *next, *owner;
    uint32_t* committed;
    uint8_t* merged;
    uint32_t cursor;
    /* online lists (tail_packed of ivf_index.hpp:115-128 split into fields) */
    uint64_t* len;
    int32_t *head, *tail;
    uint32_t* nblocks;
    uint8_t* fail;
    /* id bookkeeping (ivf_index.cpp:107-141) */
    int64_t next_id, offline_end;
    int64_t* ranges; /* [begin,end) pairs */
    uint64_t nranges, ranges_cap;
    idset supplied;
    uint64_t scalars_copied;
    /* rearrangement events */
    uint64_t* events;
    uint64_t nevents, events_cap;
};

/* ---------------------------------------------------------------- distance */

float orc_l2_sqr(const float* a, const float* b, uint32_t dim) {
    float acc = 0.0f;
    for (uint32_t d = 0; d < dim; ++d) {
        const float t = a[d] - b[d];
        const float sq = t * t;
        acc = acc + sq;
    }
    return acc;
}

float orc_l2_sqr_strided(const float* q, const float* base, uint32_t stride, uint32_t dim) {
    float acc = 0.0f;
    for (uint32_t d = 0; d < dim; ++d) {
        const float t = q[d] - base[(uint64_t)d * stride];
        const float sq = t * t;
        acc = acc + sq;
    }
    return acc;
}

float orc_ip(const float* a, const float* b, uint32_t dim) {
    float acc = 0.0f;
    for (uint32_t d = 0; d < dim; ++d) {
        const float p = a[d] * b[d];
        acc = acc + p;
    }
    return acc;
}

static float orc_ip_strided(const float* q, const float* base, uint32_t stride, uint32_t dim) {
    float acc = 0.0f;
    for (uint32_t d = 0; d < dim; ++d) {
        const float p = q[d] * base[(uint64_t)d * stride];
        acc = acc + p;
    }
    return acc;
}

uint64_t orc_interleaved_offset(uint64_t slot, uint64_t d, uint64_t dim, uint64_t group) {
    return (slot / group) * group * dim + d * group + (slot % group);
}

/* Ranking key: L2 -> squared distance; IP -> -s so ascending order ranks by
 * descending inner product. */
static float key_contig(const orc_index* h, const float* q, const float* x) {
    return h->metric == ORC_IP ? -orc_ip(q, x, h->D) : orc_l2_sqr(q, x, h->D);
}
static float key_strided(const orc_index* h, const float* q, const float* base) {
    return h->metric == ORC_IP ? -orc_ip_strided(q, base, h->G, h->D)
                               : orc_l2_sqr_strided(q, base, h->G, h->D);
}

/* ---------------------------------------------------------------- helpers */

static void* xcalloc(uint64_t n, uint64_t sz) {
    void* p = calloc(n ? n : 1, sz ? sz : 1);
    if (!p) abort();
    return p;
}

static uint64_t hash64(int64_t k) {
    uint64_t x = (uint64_t)k;
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdULL;
    x ^= x >> 33;
    x *= 0xc4ceb9fe1a85ec53ULL;
    x ^= x >> 33;
    return x;
}

/* returns 1 if newly inserted, 0 if present (keys are >= 0; -1 marks empty) */
static int idset_insert(idset* s, int64_t k) {
    if ((s->used + 1) * 2 > s->cap) {
        uint64_t ncap = s->cap ? s->cap * 2 : 64;
        int64_t* nk = (int64_t*)xcalloc(ncap, sizeof(int64_t));
        for (uint64_t i = 0; i < ncap; ++i) nk[i] = -1;
        for (uint64_t i = 0; i < s->cap; ++i) {
            if (s->keys[i] < 0) continue;
            uint64_t j = hash64(s->keys[i]) & (ncap - 1);
            while (nk[j] >= 0) j = (j + 1) & (ncap - 1);
            nk[j] = s->keys[i];
        }
        free(s->keys);
        s->keys = nk;
        s->cap = ncap;
    }
    uint64_t j = hash64(k) & (s->cap - 1);
    while (s->keys[j] >= 0) {
        if (s->keys[j] == k) return 0;
        j = (j + 1) & (s->cap - 1);
    }
    s->keys[j] = k;
    s->used++;
    return 1;
}

/* ---------------------------------------------------------------- top-k */

/* topk.hpp:14-43: keep the k smallest (dist, id) pairs, lexicographic, so
 * equal distances resolve by ascending id; result ascending, length
 * min(k, pushed).  Kept as a sorted array (insertion), same result set. */
typedef struct {
    uint64_t k, n;
    float* d;
    int64_t* id;
} topk;

static int pair_less(float da, int64_t ia, float db, int64_t ib) {
    return da < db || (da == db && ia < ib);
}

static void topk_push(topk* t, float d, int64_t id) {
    if (t->n == t->k && !pair_less(d, id, t->d[t->n - 1], t->id[t->n - 1])) return;
    uint64_t pos = t->n < t->k ? t->n : t->k - 1;
    while (pos > 0 && pair_less(d, id, t->d[pos - 1], t->id[pos - 1])) {
        t->d[pos] = t->d[pos - 1];
        t->id[pos] = t->id[pos - 1];
        --pos;
    }
    t->d[pos] = d;
    t->id[pos] = id;
    if (t->n < t->k) t->n++;
}

/* ---------------------------------------------------------------- lifecycle */

orc_index* orc_create(uint32_t num_clusters, uint32_t dim, uint32_t block_capacity,
                      uint32_t num_blocks, uint32_t interleave_group,
                      uint64_t rearrange_threshold, int metric) {
    if (num_clusters < 1 || dim < 1 || block_capacity < 1 || num_blocks < 1 ||
        interleave_group < 1)
        return NULL;
    orc_index* h = (orc_index*)xcalloc(1, sizeof(orc_index));
    h->C = num_clusters;
    h->D = dim;
    h->T = block_capacity;
    h->G = interleave_group;
    h->nblk_total = num_blocks;
    h->metric = (uint32_t)metric;
    h->threshold = rearrange_threshold;
    /* block_store.hpp:27-32 */
    h->groups_per_block = (block_capacity + interleave_group - 1) / interleave_group;
    h->payload_scalars = h->groups_per_block * interleave_group * dim;
    h->centroids = (float*)xcalloc((uint64_t)num_clusters * dim, sizeof(float));
    h->off_count = (uint64_t*)xcalloc(num_clusters, sizeof(uint64_t));
    h->off_ids = (int64_t**)xcalloc(num_clusters, sizeof(int64_t*));
    h->off_pay = (float**)xcalloc(num_clusters, sizeof(float*));
    /* block_store.cpp:19-29: zero-filled arena, ids -1, empty headers */
    h->arena = (float*)xcalloc((uint64_t)num_blocks * h->payload_scalars, sizeof(float));
    h->bids = (int64_t*)xcalloc((uint64_t)num_blocks * block_capacity, sizeof(int64_t));
    for (uint64_t i = 0; i < (uint64_t)num_blocks * block_capacity; ++i) h->bids[i] = -1;
    h->prev = (int32_t*)xcalloc(num_blocks, sizeof(int32_t));
    h->next = (int32_t*)xcalloc(num_blocks, sizeof(int32_t));
    h->owner = (int32_t*)xcalloc(num_blocks, sizeof(int32_t));
    for (uint32_t b = 0; b < num_blocks; ++b) h->prev[b] = h->next[b] = h->owner[b] = -1;
    h->committed = (uint32_t*)xcalloc(num_blocks, sizeof(uint32_t));
    h->merged = (uint8_t*)xcalloc(num_blocks, 1);
    h->len = (uint64_t*)xcalloc(num_clusters, sizeof(uint64_t));
    h->head = (int32_t*)xcalloc(num_clusters, sizeof(int32_t));
    h->tail = (int32_t*)xcalloc(num_clusters, sizeof(int32_t));
    for (uint32_t c = 0; c < num_clusters; ++c) h->head[c] = h->tail[c] = -1;
    h->nblocks = (uint32_t*)xcalloc(num_clusters, sizeof(uint32_t));
    h->fail = (uint8_t*)xcalloc(num_clusters, 1);
    return h;
}

void orc_destroy(orc_index* h) {
    if (!h) return;
    for (uint32_t c = 0; c < h->C; ++c) {
        free(h->off_ids[c]);
        free(h->off_pay[c]);
    }
    free(h->off_ids);
    free(h->off_pay);
    free(h->off_count);
    free(h->centroids);
    free(h->arena);
    free(h->bids);
    free(h->prev);
    free(h->next);
    free(h->owner);
    free(h->committed);
    free(h->merged);
    free(h->len);
    free(h->head);
    free(h->tail);
    free(h->nblocks);
    free(h->fail);
    free(h->ranges);
    free(h->supplied.keys);
    free(h->events);
    free(h);
}

void orc_set_centroids(orc_index* h, const float* centroids) {
    memcpy(h->centroids, centroids, (uint64_t)h->C * h->D * sizeof(float));
}

/* ivf_index.cpp:61-82: counts per cluster, then each row appended to its
 * cluster's segment in ascending row order, payload padded to whole groups.
 * next_id / offline_ids_end = n (ivf_index.cpp:57-58).  With explicit ids
 * (sharded load) the ids are recorded as supplied instead. */
int orc_bulk_load(orc_index* h, const float* x, uint64_t n, const uint32_t* assignment,
                  const int64_t* ids) {
    const uint64_t D = h->D, G = h->G;
    uint64_t* counts = (uint64_t*)xcalloc(h->C, sizeof(uint64_t));
    for (uint64_t i = 0; i < n; ++i) {
        if (assignment[i] >= h->C) {
            free(counts);
            return ORC_EINVAL;
        }
        counts[assignment[i]]++;
    }
    for (uint32_t c = 0; c < h->C; ++c) {
        free(h->off_ids[c]);
        free(h->off_pay[c]);
        const uint64_t groups = (counts[c] + G - 1) / G;
        h->off_ids[c] = (int64_t*)xcalloc(counts[c], sizeof(int64_t));
        h->off_pay[c] = (float*)xcalloc(groups * G * D, sizeof(float));
        h->off_count[c] = 0;
    }
    for (uint64_t i = 0; i < n; ++i) {
        const uint32_t c = assignment[i];
        const uint64_t slot = h->off_count[c]++;
        h->off_ids[c][slot] = ids ? ids[i] : (int64_t)i;
        float* base = h->off_pay[c] + orc_interleaved_offset(slot, 0, D, G);
        for (uint64_t d = 0; d < D; ++d) base[d * G] = x[i * D + d];
    }
    free(counts);
    if (ids) {
        int64_t mx = -1;
        for (uint64_t i = 0; i < n; ++i) {
            idset_insert(&h->supplied, ids[i]);
            if (ids[i] > mx) mx = ids[i];
        }
        if (mx + 1 > h->next_id) h->next_id = mx + 1;
    } else {
        h->next_id = (int64_t)n;
        h->offline_end = (int64_t)n;
    }
    return ORC_OK;
}

/* ---------------------------------------------------------------- quantizer */

/* ivf_index.cpp:93-105: argmin over clusters, strict '<' keeps the lowest
 * cluster id on ties. */
uint32_t orc_assign(const orc_index* h, const float* y) {
    float best = INFINITY;
    uint32_t best_c = 0;
    for (uint32_t c = 0; c < h->C; ++c) {
        const float k = key_contig(h, y, h->centroids + (uint64_t)c * h->D);
        if (k < best) {
            best = k;
            best_c = c;
        }
    }
    return best_c;
}

/* ivf_index.cpp:271-276: all centroid keys, then the first nprobe under
 * (key, cluster id) lexicographic order (partial_sort on pairs). */
int orc_probes(const orc_index* h, const float* q, uint64_t nprobe, uint32_t* out) {
    if (nprobe < 1 || nprobe > h->C) return ORC_EINVAL;
    topk t = {nprobe, 0, (float*)xcalloc(nprobe, sizeof(float)),
              (int64_t*)xcalloc(nprobe, sizeof(int64_t))};
    for (uint32_t c = 0; c < h->C; ++c)
        topk_push(&t, key_contig(h, q, h->centroids + (uint64_t)c * h->D), c);
    for (uint64_t p = 0; p < nprobe; ++p) out[p] = (uint32_t)t.id[p];
    free(t.d);
    free(t.id);
    return ORC_OK;
}

/* ---------------------------------------------------------------- pool */

static float* slot_base(orc_index* h, int32_t b, uint64_t slot) {
    return h->arena + (uint64_t)b * h->payload_scalars +
           orc_interleaved_offset(slot, 0, h->D, h->G);
}

/* Block `mid` of cluster c's online list, in logical order. */
static int32_t list_block(const orc_index* h, uint32_t c, uint64_t mid) {
    int32_t b = h->head[c];
    for (uint64_t i = 0; i < mid && b >= 0; ++i) b = h->next[b];
    return b;
}

/* ---------------------------------------------------------------- insert */

/* ivf_index.cpp:107-120 */
static int is_duplicate_id(orc_index* h, int64_t id) {
    if (id < 0) return 1;
    if (id < h->offline_end) return 1;
    for (uint64_t r = 0; r < h->nranges; ++r)
        if (id >= h->ranges[2 * r] && id < h->ranges[2 * r + 1]) return 1;
    if (!idset_insert(&h->supplied, id)) return 1;
    if (id >= h->next_id) h->next_id = id + 1;
    return 0;
}

/* ivf_index.cpp:166-215 (place_vector) + block_store.cpp:31-90.  Sequential
 * equivalent of the designated-writer protocol: slot did = length++, block
 * mid = did / T_m.  A block is allocated when mid reaches the list's block
 * count (with no deletes that is exactly moff == 0); a poisoned list or an
 * exhausted pool fails the vector and rolls length back.  With deletes an
 * emptied tail block stays linked and is reused. */
static int place_vector(orc_index* h, uint32_t c, const float* y, int64_t id) {
    const uint64_t did = h->len[c];
    const uint64_t mid = did / h->T, moff = did % h->T;
    int32_t b;
    if (mid >= h->nblocks[c]) {
        if (h->fail[c]) return 0;
        if (h->cursor >= h->nblk_total) { /* block_store.cpp:35: no index consumed */
            h->fail[c] = 1;
            return 0;
        }
        b = (int32_t)h->cursor++;
        h->owner[b] = (int32_t)c;
        if (h->nblocks[c] == 0) {
            h->head[c] = b;
        } else { /* block_store.cpp:55-65 link_blocks */
            h->next[h->tail[c]] = b;
            h->prev[b] = h->tail[c];
        }
        h->tail[c] = b;
        h->nblocks[c]++;
    } else {
        b = list_block(h, c, mid);
    }
    h->len[c] = did + 1;
    /* block_store.cpp:67-81 write_slot (interleaved scatter) */
    h->bids[(uint64_t)b * h->T + moff] = id;
    float* base = slot_base(h, b, moff);
    for (uint32_t d = 0; d < h->D; ++d) base[(uint64_t)d * h->G] = y[d];
    h->scalars_copied += h->D;
    /* block_store.cpp:83-90 publish_slot: prefix commit */
    h->committed[b] = (uint32_t)(moff + 1);
    return 1;
}

/* ivf_index.cpp:122-164 */
int orc_insert(orc_index* h, const float* x, uint64_t n, const int64_t* ids, int64_t* out_ids,
               uint64_t* inserted) {
    *inserted = 0;
    for (uint64_t i = 0; i < n; ++i) out_ids[i] = -1;
    if (n == 0) return ORC_OK;
    int64_t base = -1;
    if (!ids) {
        base = h->next_id;
        h->next_id += (int64_t)n;
        if (h->nranges > 0 && h->ranges[2 * (h->nranges - 1) + 1] == base) {
            h->ranges[2 * (h->nranges - 1) + 1] = base + (int64_t)n;
        } else {
            if (h->nranges == h->ranges_cap) {
                h->ranges_cap = h->ranges_cap ? 2 * h->ranges_cap : 8;
                h->ranges = (int64_t*)realloc(h->ranges, 2 * h->ranges_cap * sizeof(int64_t));
            }
            h->ranges[2 * h->nranges] = base;
            h->ranges[2 * h->nranges + 1] = base + (int64_t)n;
            h->nranges++;
        }
    }
    int exhausted = 0;
    for (uint64_t i = 0; i < n; ++i) {
        int64_t id;
        if (!ids) {
            id = base + (int64_t)i;
        } else {
            id = ids[i];
            if (is_duplicate_id(h, id)) continue;
        }
        const float* y = x + i * h->D;
        const uint32_t c = orc_assign(h, y);
        if (place_vector(h, c, y, id)) {
            out_ids[i] = id;
            (*inserted)++;
        } else {
            exhausted = 1;
        }
    }
    return exhausted ? ORC_EPOOL : ORC_OK;
}

/* ---------------------------------------------------------------- search */

/* ivf_index.cpp:262-298: validate, probe, then for each probe the offline
 * segment and the online list in block order, all into one TopK. */
int orc_search(const orc_index* h, const float* q, uint64_t k, uint64_t nprobe,
               int64_t* out_ids, float* out_d, uint64_t* count) {
    *count = 0;
    if (k < 1 || nprobe < 1 || nprobe > h->C) return ORC_EINVAL;
    uint32_t* probes = (uint32_t*)xcalloc(nprobe, sizeof(uint32_t));
    orc_probes(h, q, nprobe, probes);
    topk t = {k, 0, out_d, out_ids};
    for (uint64_t p = 0; p < nprobe; ++p) {
        const uint32_t c = probes[p];
        for (uint64_t i = 0; i < h->off_count[c]; ++i)
            topk_push(&t, key_strided(h, q, h->off_pay[c] + orc_interleaved_offset(i, 0, h->D, h->G)),
                      h->off_ids[c][i]);
        uint64_t visited = 0;
        for (int32_t b = h->head[c]; b >= 0; b = h->next[b]) {
            if (++visited > h->nblk_total) break;
            for (uint32_t s = 0; s < h->committed[b]; ++s)
                topk_push(&t,
                          key_strided(h, q, h->arena + (uint64_t)b * h->payload_scalars +
                                                orc_interleaved_offset(s, 0, h->D, h->G)),
                          h->bids[(uint64_t)b * h->T + s]);
        }
    }
    *count = t.n;
    free(probes);
    return ORC_OK;
}

/* ---------------------------------------------------------------- rearrange */

/* ivf_index.cpp:300-311 — Eq. 3, strictly greater */
int orc_exceed(const orc_index* h, uint32_t c) {
    uint64_t sum = 0, visited = 0;
    for (int32_t b = h->head[c]; b >= 0; b = h->next[b]) {
        if (++visited > h->nblk_total) return -1;
        sum += h->committed[b];
    }
    return sum > h->threshold ? 1 : 0;
}

typedef struct {
    uint32_t* q;
    uint64_t head, n, cap;
    uint8_t* queued;
} workq;

static void wq_push(workq* w, uint32_t c) {
    if (w->queued[c]) return;
    w->queued[c] = 1;
    w->q[(w->head + w->n) % w->cap] = c;
    w->n++;
}

/* ivf_index.cpp:356-368 (remap_cluster_refs) */
static void remap_refs(orc_index* h, int32_t c, int32_t a, int32_t b) {
    if (h->head[c] == a) h->head[c] = b;
    else if (h->head[c] == b) h->head[c] = a;
    if (h->tail[c] == a) h->tail[c] = b;
    else if (h->tail[c] == b) h->tail[c] = a;
}

static int32_t remap1(int32_t x, int32_t a, int32_t b) { return x == a ? b : (x == b ? a : x); }

/* ivf_index.cpp:370-412 (swap_blocks): exchange the contents (ids, payload, committed) of
 * physical blocks a and b, then rewrite both headers and every neighbour /
 * list-head / list-tail reference so both logical lists are unchanged. */
static void swap_blocks(orc_index* h, int32_t a, int32_t b) {
    if (a == b) return;
    const int32_t pa = h->prev[a], na = h->next[a], pb = h->prev[b], nb = h->next[b];
    const int32_t oa = h->owner[a], ob = h->owner[b];
    {
        float* A = h->arena + (uint64_t)a * h->payload_scalars;
        float* B = h->arena + (uint64_t)b * h->payload_scalars;
        for (uint64_t i = 0; i < h->payload_scalars; ++i) {
            const float t = A[i];
            A[i] = B[i];
            B[i] = t;
        }
        int64_t* IA = h->bids + (uint64_t)a * h->T;
        int64_t* IB = h->bids + (uint64_t)b * h->T;
        for (uint32_t i = 0; i < h->T; ++i) {
            const int64_t t = IA[i];
            IA[i] = IB[i];
            IB[i] = t;
        }
        const uint32_t t = h->committed[a];
        h->committed[a] = h->committed[b];
        h->committed[b] = t;
    }
    h->prev[a] = remap1(pb, a, b);
    h->next[a] = remap1(nb, a, b);
    h->owner[a] = ob;
    h->prev[b] = remap1(pa, a, b);
    h->next[b] = remap1(na, a, b);
    h->owner[b] = oa;
    h->merged[a] = 0;
    h->merged[b] = 0;
    if (pa >= 0 && pa != a && pa != b) h->next[pa] = b;
    if (na >= 0 && na != a && na != b) h->prev[na] = b;
    if (pb >= 0 && pb != a && pb != b) h->next[pb] = a;
    if (nb >= 0 && nb != a && nb != b) h->prev[nb] = a;
    if (oa >= 0) remap_refs(h, oa, a, b);
    if (ob >= 0 && ob != oa) remap_refs(h, ob, a, b);
}

/* ivf_index.cpp:414-434 (split_runs_around): break fused runs touching x; owners re-merge later */
static void split_runs_around(orc_index* h, int32_t x, workq* w) {
    if (h->merged[x]) {
        h->merged[x] = 0;
        if (h->owner[x] >= 0) wq_push(w, (uint32_t)h->owner[x]);
    }
    const int32_t nx = h->next[x];
    if (nx >= 0 && h->merged[nx]) {
        h->merged[nx] = 0;
        if (h->owner[x] >= 0) wq_push(w, (uint32_t)h->owner[x]);
    }
}

/* ivf_index.cpp:436-474 (rearrange_locked) (Alg. 3): walk the list; for every logical link u->v
 * that is not fused, pull v into the physical successor p = u+1 (swap), or
 * just mark the fusion when v already is u+1. */
static void rearrange_list(orc_index* h, uint32_t c, uint64_t* merges, workq* w) {
    const uint32_t allocated = h->cursor;
    int32_t u = h->head[c];
    if (u < 0) return;
    const uint64_t cap = 4ull * allocated + 64;
    for (uint64_t guard = 0; guard < cap; ++guard) {
        const int32_t v = h->next[u];
        if (v < 0) break;
        if (h->merged[v]) {
            u = v;
            continue;
        }
        const int32_t p = u + 1;
        if ((uint32_t)p >= allocated) {
            u = v;
            continue;
        }
        if (p == v) {
            h->merged[v] = 1;
            (*merges)++;
            u = v;
            continue;
        }
        split_runs_around(h, p, w);
        split_runs_around(h, v, w);
        swap_blocks(h, p, v);
        h->merged[p] = 1;
        (*merges)++;
        u = p;
    }
}

/* ivf_index.cpp:476-505: work queue seeded with c, displaced owners
 * re-merged lazily, bounded by 2C+8 rounds; one event per call. */
int orc_rearrange(orc_index* h, uint32_t c) {
    if (c >= h->C) return ORC_ERANGE;
    const uint64_t hops_before = orc_hop_count(h, c);
    workq w = {(uint32_t*)xcalloc(h->C, sizeof(uint32_t)), 0, 0, h->C,
               (uint8_t*)xcalloc(h->C, 1)};
    wq_push(&w, c);
    uint64_t merges = 0, rounds = 0;
    while (w.n > 0 && rounds++ < 2ull * h->C + 8) {
        const uint32_t x = w.q[w.head];
        w.head = (w.head + 1) % w.cap;
        w.n--;
        w.queued[x] = 0;
        rearrange_list(h, x, &merges, &w);
    }
    free(w.q);
    free(w.queued);
    if (h->nevents == h->events_cap) {
        h->events_cap = h->events_cap ? 2 * h->events_cap : 16;
        h->events = (uint64_t*)realloc(h->events, 4 * h->events_cap * sizeof(uint64_t));
    }
    uint64_t* e = h->events + 4 * h->nevents++;
    e[0] = c;
    e[1] = hops_before;
    e[2] = orc_hop_count(h, c);
    e[3] = merges;
    return ORC_OK;
}

/* ivf_index.cpp:507-511 */
int orc_rearrange_sweep(orc_index* h) {
    for (uint32_t c = 0; c < h->C; ++c) {
        const int e = orc_exceed(h, c);
        if (e < 0) return ORC_ECORRUPT;
        if (e) orc_rearrange(h, c);
    }
    return ORC_OK;
}

uint64_t orc_take_events(orc_index* h, uint64_t* out4, uint64_t cap) {
    uint64_t n = h->nevents < cap ? h->nevents : cap;
    memcpy(out4, h->events, 4 * n * sizeof(uint64_t));
    h->nevents = 0;
    return n;
}

/* ---------------------------------------------------------------- delete */

/* Extension (the reference has no delete).  Requests are
 * applied in ascending request order.  A hole is filled by the LAST vector
 * of the same part (offline segment, or the online list's last committed
 * slot), which then shrinks by one: tail block committed - 1 and length - 1.
 * Blocks are never returned to the pool; an emptied tail block stays linked
 * (and is reused by the next insert).  A vacated online slot gets id -1; its
 * payload is left as is.  Unknown ids are reported via found[i] = 0. */
int orc_remove(orc_index* h, const int64_t* ids, uint64_t n, uint64_t* removed, uint8_t* found) {
    *removed = 0;
    const uint64_t D = h->D, G = h->G;
    for (uint64_t r = 0; r < n; ++r) {
        const int64_t id = ids[r];
        int done = 0;
        for (uint32_t c = 0; c < h->C && !done; ++c) {
            for (uint64_t i = 0; i < h->off_count[c]; ++i) {
                if (h->off_ids[c][i] != id) continue;
                const uint64_t last = h->off_count[c] - 1;
                if (i != last) {
                    h->off_ids[c][i] = h->off_ids[c][last];
                    float* dst = h->off_pay[c] + orc_interleaved_offset(i, 0, D, G);
                    const float* src = h->off_pay[c] + orc_interleaved_offset(last, 0, D, G);
                    for (uint64_t d = 0; d < D; ++d) dst[d * G] = src[d * G];
                }
                h->off_count[c] = last;
                done = 1;
                break;
            }
            if (done) break;
            uint64_t did = 0;
            for (int32_t b = h->head[c]; b >= 0 && !done; b = h->next[b]) {
                for (uint32_t s = 0; s < h->committed[b]; ++s, ++did) {
                    if (h->bids[(uint64_t)b * h->T + s] != id) continue;
                    const uint64_t last = h->len[c] - 1;
                    const int32_t lb = list_block(h, c, last / h->T);
                    const uint32_t ls = (uint32_t)(last % h->T);
                    if (did != last) {
                        h->bids[(uint64_t)b * h->T + s] = h->bids[(uint64_t)lb * h->T + ls];
                        float* dst = slot_base(h, b, s);
                        const float* src = slot_base(h, lb, ls);
                        for (uint64_t d = 0; d < D; ++d) dst[d * G] = src[d * G];
                    }
                    h->bids[(uint64_t)lb * h->T + ls] = -1;
                    h->committed[lb] = ls;
                    h->len[c] = last;
                    done = 1;
                    break;
                }
            }
        }
        if (found) found[r] = (uint8_t)done;
        if (done) (*removed)++;
    }
    return ORC_OK;
}

/* ---------------------------------------------------------------- introspection */

uint64_t orc_size(const orc_index* h) {
    uint64_t t = 0;
    for (uint32_t c = 0; c < h->C; ++c) t += h->off_count[c] + h->len[c];
    return t;
}
uint64_t orc_scalars_copied(const orc_index* h) { return h->scalars_copied; }
uint64_t orc_list_length(const orc_index* h, uint32_t c) { return h->len[c]; }
uint64_t orc_offline_count(const orc_index* h, uint32_t c) { return h->off_count[c]; }
int32_t orc_online_head(const orc_index* h, uint32_t c) { return h->head[c]; }
uint32_t orc_online_blocks(const orc_index* h, uint32_t c) { return h->nblocks[c]; }
uint64_t orc_allocated_blocks(const orc_index* h) { return h->cursor; }
int64_t orc_next_id(const orc_index* h) { return h->next_id; }

/* block_store.cpp:111-132: a hop is a next link whose target is not fused */
uint64_t orc_hop_count(const orc_index* h, uint32_t c) {
    uint64_t hops = 0, visited = 0;
    for (int32_t b = h->head[c]; b >= 0; b = h->next[b]) {
        if (++visited > h->nblk_total) return UINT64_MAX;
        const int32_t nx = h->next[b];
        if (nx >= 0 && !h->merged[nx]) hops++;
    }
    return hops;
}

void orc_block_header(const orc_index* h, int32_t b, int32_t* out5) {
    out5[0] = h->prev[b];
    out5[1] = h->next[b];
    out5[2] = (int32_t)h->committed[b];
    out5[3] = h->owner[b];
    out5[4] = h->merged[b];
}
void orc_block_ids(const orc_index* h, int32_t b, int64_t* out) {
    memcpy(out, h->bids + (uint64_t)b * h->T, h->T * sizeof(int64_t));
}
void orc_block_payload(const orc_index* h, int32_t b, float* out) {
    memcpy(out, h->arena + (uint64_t)b * h->payload_scalars, h->payload_scalars * sizeof(float));
}
void orc_offline_segment(const orc_index* h, uint32_t c, int64_t* ids, float* payload) {
    const uint64_t n = h->off_count[c];
    memcpy(ids, h->off_ids[c], n * sizeof(int64_t));
    const uint64_t groups = (n + h->G - 1) / h->G;
    memcpy(payload, h->off_pay[c], groups * h->G * h->D * sizeof(float));
}

/* ivf_index.cpp:334-354 (cluster_contents): offline then online (traverse order) */
uint64_t orc_cluster_contents(const orc_index* h, uint32_t c, int64_t* ids, float* vecs) {
    uint64_t n = 0;
    const uint64_t D = h->D, G = h->G;
    for (uint64_t i = 0; i < h->off_count[c]; ++i, ++n) {
        if (!ids) continue;
        ids[n] = h->off_ids[c][i];
        const float* base = h->off_pay[c] + orc_interleaved_offset(i, 0, D, G);
        for (uint64_t d = 0; d < D; ++d) vecs[n * D + d] = base[d * G];
    }
    uint64_t visited = 0;
    for (int32_t b = h->head[c]; b >= 0; b = h->next[b]) {
        if (++visited > h->nblk_total) break;
        for (uint32_t s = 0; s < h->committed[b]; ++s, ++n) {
            if (!ids) continue;
            ids[n] = h->bids[(uint64_t)b * h->T + s];
            const float* base = h->arena + (uint64_t)b * h->payload_scalars +
                                orc_interleaved_offset(s, 0, D, G);
            for (uint64_t d = 0; d < D; ++d) vecs[n * D + d] = base[d * G];
        }
    }
    return n;
}
