// Error plumbing for the C ABI (thread-local last error) and the pinned synthetic-token
// convention shared by the executor, the stage and the CPU oracle.
#pragma once

#include <cstdint>
#include <string>

#include "deserve.h"

// Records msg as the thread's last error and returns code.
int32_t ds_fail(int32_t code, const std::string& msg);

constexpr int32_t kBosToken = 128000;
constexpr int32_t kPromptVocab = 128000;

inline uint64_t ds_splitmix(uint64_t z) {
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

inline int32_t ds_prompt_token(int64_t req_id, int32_t pos) {
    if (pos == 0) return kBosToken;
    const uint64_t h = ds_splitmix(0x5EEDULL ^ (uint64_t(req_id) * 0x9E3779B97F4A7C15ULL) ^
                                   uint64_t(pos));
    return int32_t(h % uint64_t(kPromptVocab));
}
