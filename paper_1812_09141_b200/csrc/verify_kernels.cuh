// verify_kernels.cuh -- the sm_100a verification kernels (declarations + launch params).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "ssj_device.cuh"

namespace ssjb {

// Geometry of the warp-tile kernel (strategy A, short slices): every warp owns
// kTile = 32 * SSJB_TILE_ITEMS consecutive slots.
#ifndef SSJB_TILE_THREADS
#define SSJB_TILE_THREADS 128
#endif
#ifndef SSJB_TILE_ITEMS
#define SSJB_TILE_ITEMS 2
#endif
#ifndef SSJB_TILE_MIN_BLOCKS
#define SSJB_TILE_MIN_BLOCKS 8
#endif
constexpr uint32_t kThreadsA = SSJB_TILE_THREADS;            // threads per CTA
constexpr uint32_t kTile = 32 * SSJB_TILE_ITEMS;             // slots per warp tile
constexpr int kTileMinBlocks = SSJB_TILE_MIN_BLOCKS;         // CTAs per SM (register cap)
#ifndef SSJB_BM_MIN_CANDS
#define SSJB_BM_MIN_CANDS 64
#endif
constexpr uint32_t kSliceBitmapMinCands = SSJB_BM_MIN_CANDS;  // slices this long get a probe bitmap per chunk
constexpr uint32_t kMaxBitmapWords = 8192;     // probe token range cap (256K tokens)
constexpr uint32_t kNone = 0xFFFFFFFFu;
#ifndef SSJB_LONG_PAIR
#define SSJB_LONG_PAIR 160
#endif
constexpr uint32_t kLongPair = SSJB_LONG_PAIR;  // candidates longer than this: long_slice_kernel

// Strategy A, long slices ("runs"): a run is a piece of <= kRun consecutive slots of one
// slice with >= kRunMinSlice candidates (slices are cut at the chunk-segment boundaries
// first). run_kernel verifies runs with the probe bitmap staged in shared memory; every
// other slot (short slices, uncovered slots) is verified by warp_tile_kernel over a list of
// tiles.
#ifndef SSJB_RUN_MIN_SLICE
#define SSJB_RUN_MIN_SLICE 128
#endif
#ifndef SSJB_RUN_MIN_BLOCKS
#define SSJB_RUN_MIN_BLOCKS 4
#endif
#ifndef SSJB_RUN_BLOCK
#define SSJB_RUN_BLOCK 16
#endif
#ifndef SSJB_RUN_MAP_BITS
#define SSJB_RUN_MAP_BITS 0  // 1: the probe map in shared memory is a bitmap (slower: ALU)
#endif
#ifndef SSJB_RUN_THREADS
#define SSJB_RUN_THREADS 256
#endif
#ifndef SSJB_RUN_ITEMS
#define SSJB_RUN_ITEMS 2
#endif
constexpr uint32_t kRunThreads = SSJB_RUN_THREADS;
constexpr uint32_t kRunItems = SSJB_RUN_ITEMS;          // slots per thread per run
constexpr uint32_t kRun = kRunThreads * kRunItems;      // slots per run
constexpr uint32_t kRunMinSlice = SSJB_RUN_MIN_SLICE;
constexpr uint32_t kRunMapRange = 8160;                 // probe token range held as a byte map
constexpr uint32_t kRunMapBytes = 8192;                 // byte map (range + empty entry)
constexpr uint32_t kRunMapWords = kRunMapRange / 32 + 1;  // the probe's bitmap words / ranks
constexpr uint32_t kRunMapBuf = kRunMapBytes + 2 * ((kRunMapWords + 3) & ~3u) * 4;
constexpr int kRunMinBlocks = SSJB_RUN_MIN_BLOCKS;
constexpr uint32_t kRunBlock = SSJB_RUN_BLOCK;          // consecutive runs per CTA turn
// shared memory: two candidate-head buffers per warp [buf][item][lane] 32 bytes (the
// current one doubles as the warp's continuation queue), two or three probe byte maps
#ifndef SSJB_RUN_HEAD_BUFS
#define SSJB_RUN_HEAD_BUFS 0
#endif
constexpr uint32_t kRunHeadBufs = SSJB_RUN_HEAD_BUFS;  // 2: heads of run k+1 fetched during run k
// probe-map buffers: 2, or 3 when slices are short (maps change every run or two, and one
// warp builds the next map while the others still verify: run_kernel's build-ahead)
#ifndef SSJB_RUN_MB3_BELOW
#define SSJB_RUN_MB3_BELOW 2048  // average candidates per slice below which 3 buffers are used
#endif
constexpr size_t run_smem_bytes(uint32_t map_bufs) {
    // per warp: the continuation queue (I*32 entries of 16 bytes), or with cp.async head
    // buffers (kRunHeadBufs > 0) that many buffers of I*64 uint4
    return (size_t)(kRunThreads / 32) * 16 *
               (kRunHeadBufs ? (size_t)kRunHeadBufs * kRunItems * 64 : (size_t)kRunItems * 32) +
           map_bufs * kRunMapBuf;
}

struct RunDesc {
    uint32_t slice;  // slice index
    uint32_t begin;  // first slot
    uint32_t end;    // one past the last slot
    uint32_t pad;
};

// Per-slice descriptor built once per chunk by prep_kernel (32 bytes, one sector).
struct SliceDesc {
    uint32_t end;     // cumulative end offset in C
    uint32_t rpos8;   // probe set position (8-token units)
    uint32_t rsize;   // |r|
    uint32_t bofs;    // probe bitmap (bm_bits / bm_rank word offset) or kNone
    uint32_t lo;      // bitmap base token (multiple of 32)
    uint32_t nwords;  // bitmap words
    uint32_t pad0, pad1;
};

// Result-block words (SSJ_RESULT_WORDS = 8): 0 count, 1 error bits, 2..4 stats,
// 5 bitmap words allocated in this chunk, 6 slices given a bitmap.
constexpr int kAccBitmapWords = 5;
constexpr int kAccBitmapSlices = 6;  // 6: slices given a bitmap in this chunk

// Everything a verification kernel needs. Device pointers only.
struct KParams {
    const uint32_t* tokens;  // padded CSR
    const uint2* sets;       // {pos8, size}
    uint32_t n_sets;
    const uint32_t* C;       // candidate slots
    uint64_t nC;
    const uint32_t* C_O;     // (probe, end) pairs
    uint32_t n_slices;
    uint32_t* tile_first;        // [n_tiles + 1], first slice with end > t * kTile
    uint32_t n_tiles;
    PredDev pred;
    const uint4* heads;             // packed set heads, 2 x uint4 per set (nullable)
    unsigned long long heads_tex;   // linear uint4 texture over heads (0: none)
    unsigned long long tokens_tex;  // linear uint4 texture over tokens (0: none)
    uint32_t long_words;            // long pass: shared bitmap words per CTA (0: kMaxBitmapWords)
    const uint32_t* req_tab;        // Jaccard/Dice: required overlap by |r|+|s| (nullable)
    uint32_t req_tab_n;
    SliceDesc* slices;              // strategy A: per-slice descriptors (nullable otherwise)
    uint32_t* bm_bits;              // probe membership bitmaps (word = 32 tokens)
    uint32_t* bm_rank;              // probe tokens below each bitmap word
    uint64_t bm_cap;                // bitmap words available (0 = no bitmaps)
    uint32_t* bm_list;              // slices given a bitmap (count in acc[kAccBitmapSlices])
    uint32_t* defer;                // strategy A: slices with long pairs (this segment)
    unsigned long long* defer_n;    // their count (this launch's segment)
    uint64_t defer_cap;
    uint32_t seg_tag;               // chunk segment index + 1 (marks in SliceDesc::pad0)
    RunDesc* runs;                  // strategy A: runs of long slices (this segment)
    unsigned long long* runs_n;
    uint64_t runs_cap;
    uint32_t* short_tiles;          // strategy A: tiles holding short-slice / uncovered slots
    unsigned long long* short_n;
    uint64_t short_cap;
    uint8_t* flags;                 // Pairs mode (nullable)
    uint32_t* res_slots;            // results mode (nullable)
    uint32_t* res_ov;
    unsigned long long* res_n;
    uint64_t res_cap;
    unsigned long long* acc;  // SSJ_RESULT_WORDS: count, err, stats[3]
    // strategy A, whole chunk (prep_kernel; ctr_all null for B / C): the chunk is cut into
    // segments of seg_slots slots (the host path's H2D pieces; one segment on the device
    // path). Segment k's runs start at runs_all + 2 * (k * seg_slots / kTile), its short tiles
    // at short_all + k * seg_slots / kTile, its counters at ctr_all + kCounters * k (+1 runs,
    // +2 short tiles).
    uint64_t seg_slots;
    RunDesc* runs_all;
    uint32_t* short_all;
    unsigned long long* ctr_all;
    unsigned long long* lb_status;  // one segment: 1 + CTAs zeroed words (ordered run list)
};

// Per-segment counters: 0 long slices marked, 1 runs, 2 short tiles, 3 long-pass slices
// taken, 4 short tiles taken.
constexpr int kCounters = 5;

enum OutKind : int { kOutCount = 0, kOutFlags = 1, kOutResults = 2 };

// Packed set heads: one 32-byte record per set -- the set's first 8 tokens (0x00FFFFFF past
// |s|) in the low 24 bits, and in the top bytes of tokens 0..3 / 4..7 the set's CSR
// position pos8 / size |s| (little-endian). Usable when every token is < kHeadTokenLimit
// (then the padding value lies outside every probe bitmap's range).
constexpr uint32_t kHeadTokenMask = 0x00FFFFFFu;
constexpr uint32_t kHeadTokenLimit = 0x00FFFFE0u;

// Launchers (stream-ordered, no synchronisation). Return cudaGetLastError().
// Build the packed heads of a collection; *max_token receives the largest token (atomicMax).
cudaError_t launch_build_heads(const uint32_t* tokens, const uint2* sets, uint32_t n_sets,
                               uint4* heads, unsigned* max_token, cudaStream_t st);
// prep_kernel (+ bitmap_kernel when p.slices && p.bm_cap): validation, slice descriptors,
// probe bitmaps and -- strategy A -- the tile index, the runs of long slices and the short-tile
// lists of every segment. Returns the number of kernels launched through *launches.
cudaError_t launch_prep(const KParams& p, cudaStream_t st, int* launches = nullptr);
// Strategy A, first pass over the segment holding tiles [tile_begin, tile_end): run_kernel
// (long slices), warp_tile_kernel (short slices)
// (aux, fork, join: when aux is set, warp_tile_kernel runs on aux concurrently with
// run_kernel on st -- they verify disjoint slots -- and st waits for it)
#ifndef SSJB_TILES_FORK
#define SSJB_TILES_FORK 1
#endif
cudaError_t launch_tiles(const KParams& p, int out, bool stats, uint32_t tile_begin,
                         uint32_t tile_end, cudaStream_t st, cudaStream_t aux = nullptr,
                         cudaEvent_t fork = nullptr, cudaEvent_t join = nullptr);
// Strategy A, second pass: slices the first pass marked for long pairs, slots of tiles
// [tile_begin, tile_end) (CTA per slice, bitmap in shared memory, one warp per pair)
cudaError_t launch_long(const KParams& p, int out, bool stats, uint32_t tile_begin,
                        uint32_t tile_end, cudaStream_t st);
// Strategy B: block of `threads` per probe slice
cudaError_t launch_block(const KParams& p, int out, bool stats, uint32_t threads,
                         cudaStream_t st);
// Strategy C: groups of G lanes per pair, merge-path partitions with round-level exits
cudaError_t launch_path(const KParams& p, int out, uint32_t group, cudaStream_t st);
// Diagnostic streaming-read kernel (bandwidth probe)
cudaError_t launch_read_bw(const void* buf, uint64_t bytes, uint32_t reps, unsigned* sink,
                           cudaStream_t st);
// H2 on the GPU: qualifying slots (p.res_slots[0..n)) -> (r_id << 32 | s_id) original ids
cudaError_t launch_pairs(const KParams& p, const uint32_t* oid, uint64_t n,
                         unsigned long long* keys, cudaStream_t st);
// Instrumentation: algorithmic bytes under the reference loop
cudaError_t launch_bytes(const KParams& p, unsigned long long* d_bytes, cudaStream_t st);

}  // namespace ssjb
