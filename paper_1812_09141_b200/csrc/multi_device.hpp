// multi_device.hpp -- one verification engine over several GPUs.
//
// A multi-device engine is an ssj_engine whose `group` holds one ordinary engine per device.
// Every C-ABI entry point dispatches to these functions when `group` is set, so callers
// (run_join's dispatcher, the C++ drop-in, Python) use it exactly like a one-GPU engine.
#pragma once

#include <cstdint>
#include <vector>

#include "../../include/ssjoin_b200.h"

namespace ssjm {

struct Group;

// Builds the per-device engines: the collection is uploaded once to devices[0] and fanned
// out device to device over NVLink (doubling tree of peer copies). *fanout_ms: the fan-out.
int create_group(Group** out, const int32_t* devices, uint32_t n_devices, const uint32_t* tokens,
                 const uint32_t* offsets, uint32_t n_sets, const ssj_predicate* pred, int32_t mode,
                 const ssj_strategy* strategy);
void destroy_group(Group* g);
ssj_engine* first(const Group& g);
uint32_t size(const Group& g);
int devices(const Group& g, int32_t* out, uint32_t cap, uint32_t* n, double* fanout_ms);

int submit(Group& g, const uint32_t* C, uint64_t nC, const uint32_t* C_O, uint64_t nCO,
           uint8_t* flags_out, uint64_t* ticket);
int wait(Group& g, uint64_t ticket, uint64_t* count_out, ssj_stats* stats);
int verify_results(Group& g, const uint32_t* C, uint64_t nC, const uint32_t* C_O, uint64_t nCO,
                   uint32_t* slots_out, uint32_t* overlaps_out, uint64_t cap, uint64_t* n_out);
int verify_pairs(Group& g, const uint32_t* C, uint64_t nC, const uint32_t* C_O, uint64_t nCO,
                 uint32_t* pairs_out, uint32_t* overlaps_out, uint64_t cap, uint64_t* n_out,
                 int sorted, ssj_stats* stats);
int set_original_ids(Group& g, const uint32_t* original_id);
int gpu_join_shard(Group& g, int32_t algorithm, uint32_t shard, uint32_t n_shards,
                   uint64_t max_chunk_candidates, uint32_t* pairs_out, uint64_t pairs_cap,
                   uint64_t* n_pairs, ssj_gpu_join_report* report);
int set_profiling(Group& g, int enabled);
int kernel_time(Group& g, double* total_ms, uint64_t* launches);

// The slice ranges of a chunk's split (exposed for tests through ssj_multi_split).
struct Range {
    uint64_t slice_begin, slice_end;  // slices [begin, end)
    uint64_t c_lo, c_hi;              // slots [c_lo, c_hi)
};
int split_chunk(const std::vector<uint32_t>& set_sizes, uint32_t parts, const uint32_t* C_O,
                uint64_t nCO, uint64_t nC, std::vector<Range>* out);

}  // namespace ssjm
