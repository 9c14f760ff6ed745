// attn_types.h — work-list records shared by the host tile scheduler
// (dfa2c.cpp) and the sm_100a fused head-wise attention kernel.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_bf16.h>
#include <vector_types.h>

namespace dfa2k {

// One unit of the per-head tile scheduler: a PAIR of 128-row query tiles
// (lanes A and B) of one (sample, head) that share one K/V tile stream — the
// union of the two tiles' mask rows, in ascending key order — or, for Cached
// heads, a 256-row copy-back from the head cache.
struct WorkItem {
    int32_t bh;          // sample * H + head: row of the [batch*H, N, d] view
    int32_t qtile_a;     // lane A query tile
    int32_t qtile_b;     // lane B query tile, -1 when the pair is a single tile
    int32_t tile_begin;  // offset into the tile-word list (compute items)
    int32_t n_tiles;     // union length (0 for copy items)
    int32_t mask_off;    // byte offset of this head's nb*nb block mask
    int32_t flags;       // ITEM_COPY | ITEM_COMMIT | ITEM_SPLIT
    int32_t part;        // ITEM_SPLIT: partial-output slot of this chunk
    int32_t group;       // ITEM_SPLIT: split group (the original pair item)
    int32_t chunk;       // ITEM_SPLIT: chunk index within the group
    int32_t nchunk;      // ITEM_SPLIT: chunks in the group
    int32_t pad;
};

enum : int32_t {
    ITEM_COPY = 1,    // Cached head: out <- cache slot (src/dispatch.cpp:77-81)
    ITEM_COMMIT = 2,  // computed head: also store O into the cache slot (:85-88)
    ITEM_SPLIT = 4,   // one key chunk of a heavy pair; the group's last chunk combines
    ITEM_MULTI = 8,   // calibration pass: every key tile in window-band order, with
                      // snapshots of O/l written to the candidates' outputs (see below)
    ITEM_HALVES = 16, // one query tile on both lanes, each folding half of its key
                      // tiles; the lanes merge (max, sum, O) in the epilogue (d = 64)
};

// Tile word: KV tile index in bits [0,24); bit 24/25: lane A/B folds this
// tile; bit 26/27: lane A/B needs element masking (mask block size != 128 or
// a ragged tail).
constexpr uint32_t TILE_INDEX_MASK = 0x00FFFFFFu;
constexpr uint32_t TILE_NEED_A = 1u << 24;
constexpr uint32_t TILE_NEED_B = 1u << 25;
constexpr uint32_t TILE_PART_A = 1u << 26;
constexpr uint32_t TILE_PART_B = 1u << 27;
// ITEM_MULTI: after folding this tile lane A/B emits its next snapshot
// (args.snap_slots[i], i = the lane's snapshot count); at the item end the
// lane emits every remaining snapshot from its final state.
constexpr uint32_t TILE_SNAP_A = 1u << 28;
constexpr uint32_t TILE_SNAP_B = 1u << 29;
// snap_slots bit m < 15: candidate output m (map `to`, row bh + m * snap_stride);
// SNAP_ORIGINAL: the original (all-Full) output (map `tc`).
constexpr uint32_t SNAP_ORIGINAL = 1u << 15;
constexpr int MAX_SNAPS = 16;
// Per-query-tile tile-set word (dfa2c_tile_set): bit 31 = needs element masking.
constexpr uint32_t TILE_SET_PARTIAL = 0x80000000u;

// Kernel arguments (besides the three TMA tensor maps).
struct AttnArgs {
    const WorkItem* items;
    const int32_t* cta_begin;  // [gridDim.x + 1]
    const uint32_t* tiles;
    const uint8_t* masks;      // concatenated nb*nb block masks
    __nv_bfloat16* out;        // [batch*H, N, D]
    __nv_bfloat16* cache;      // layer slot array [batch*H, N, D] or null
    int32_t n;
    int32_t block;
    int32_t nb;
    float scale_log2;          // log2(e) / sqrt(d)
    long long* trace;          // debug builds (-DDFA2_TRACE=1): per-tile clock64 stamps of CTA 0
    float* part_o;             // split items: [slots][2 lanes][D][128] unnormalised O
    float* part_ml;            // split items: [slots][2 lanes][2][128] reference max, row sum
    int* counters;             // split groups: [groups][2 lanes] chunks finished (zeroed per launch)
    int32_t n_peers;           // sharded P2P launches: other ranks' out buffers (PeerMaps) to store to
    int32_t copies_last;       // every CTA's copy items form the tail of its list (the copy-tail ring)
    const int2* copy_tiles;    // copy pool: (bh, query tile) of every Cached-head tile of the launch
    int32_t n_copy_tiles;      //   (0: copies are per-CTA list items)
    int32_t row_bytes;         //   bytes per row of out / cache (d x 2)
    int* copy_ctr;             //   [2]: boxes claimed, CTAs done (zero at launch; the last CTA re-zeroes)
    int32_t snap_stride;       // ITEM_MULTI: rows of `to` between candidate outputs (= batch*H)
    int32_t n_snap;            // ITEM_MULTI: snapshots per query tile (window bands + the full row)
    uint16_t snap_slots[MAX_SNAPS];
};

// Sharded launches that assemble the layer over peer memory: the TMA maps of
// the other ranks' output buffers (opened through CUDA IPC on the NVLink
// box); every output box this rank stores goes to each of them as well.
constexpr int MAX_PEERS = 7;  // world <= 8
struct PeerMaps {
    CUtensorMap m[MAX_PEERS];
    void* ptr[MAX_PEERS];  // the same buffers as raw pointers (the copy pool's 1-D bulk stores)
};

constexpr int TILE_M = 128;  // query rows per tile (tcgen05 M)
constexpr int TILE_N = 128;  // keys per KV tile (tcgen05 N of S = Q K^T)

}  // namespace dfa2k
