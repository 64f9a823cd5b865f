// host_common.hpp -- host-side (C++) helpers shared by the candidate generators, the
// synthetic-data generator and the join driver.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/ssjoin_b200.h"

namespace ssjh {

// Thread-local error channel shared with engine.cu (ssj_last_error).
int set_error(int code, const std::string& msg);

// Read-only view of the reference CSR collection (collection.hpp:76-94).
struct CollView {
    const uint32_t* tokens = nullptr;
    const uint32_t* offsets = nullptr;
    uint32_t n = 0;
    uint32_t size(uint32_t i) const { return offsets[i + 1] - offsets[i]; }
    const uint32_t* set(uint32_t i) const { return tokens + offsets[i]; }
};

// similarity.hpp:135-164 size_bounds().min (the only bound the generators use).
uint64_t size_lower_bound(const ssj_predicate& p, uint64_t size_r);

// filters.hpp:148-159 prefix lengths (probe, index).
struct PrefixLengths {
    uint32_t probe = 1;
    uint32_t index = 1;
};
PrefixLengths prefix_lengths(const ssj_predicate& p, uint32_t size);

// filters.hpp:174-181 positional filter with current_overlap = 1.
bool positional_keep(const ssj_predicate& p, uint32_t size_r, uint32_t size_s, uint32_t pos_r,
                     uint32_t pos_s);

}  // namespace ssjh
