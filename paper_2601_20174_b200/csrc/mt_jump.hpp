// paper_2601_20174_b200/csrc/mt_jump.hpp — MT19937-64 with jump-ahead, host side.
//
// The reference draws S^(0) from one sequential std::mt19937_64 stream
// (rng.hpp:22-49, smoothing.hpp:84-92). Its state is a window of 312 words of
// a GF(2)-linear recurrence, so the window J words ahead is a fixed linear map
// of the current one: with g_J(x) = x^J mod phi(x) (phi the minimal polynomial
// of the one-word shift, degree 19937) it is the XOR of the windows at the set
// coefficients of g_J. scripts/make_mt_jump_table.py derives phi and g_J for
// J = 2^17 .. 2^40 (mt_jump_table.inc); this header applies them, so several
// host threads (host_rng.hpp) or device warps (setup_kernels.cu) can each
// produce their own slice of the SAME stream, bit for bit.
#pragma once

#include <cstdint>
#include <cstring>
#include <vector>

namespace nlsp_host {

#include "mt_jump_table.inc"

constexpr int kMtN = 312, kMtM = 156, kMtDeg = 19937;
constexpr std::uint64_t kMtA = 0xB5026F5AA96619E9ull, kMtUM = 0xFFFFFFFF80000000ull, kMtLM = 0x7FFFFFFFull;

// window at position 0: the seeding recurrence of mt19937_64
inline void mt64_seed(std::uint64_t seed, std::uint64_t* win) {
    win[0] = seed;
    for (int i = 1; i < kMtN; ++i) win[i] = 6364136223846793005ull * (win[i - 1] ^ (win[i - 1] >> 62)) + (std::uint64_t)i;
}

inline std::uint64_t mt64_temper(std::uint64_t x) {
    x ^= (x >> 29) & 0x5555555555555555ull;
    x ^= (x << 17) & 0x71D67FFFEDA60000ull;
    x ^= (x << 37) & 0xFFF7EEE000000000ull;
    x ^= x >> 43;
    return x;
}

// The generator positioned at a window: outputs temper(x[p + 312 + i]), i = 0, 1, ...
// (a freshly seeded window gives the outputs of std::mt19937_64(seed))
class Mt64 {
public:
    Mt64() = default;
    explicit Mt64(const std::uint64_t* win) { load(win); }
    void load(const std::uint64_t* win) {
        std::memcpy(mt_, win, sizeof(mt_));
        idx_ = kMtN;
    }
    std::uint64_t operator()() {
        if (idx_ >= kMtN) twist();
        return mt64_temper(mt_[idx_++]);
    }

private:
    void twist() {
        for (int i = 0; i < kMtN; ++i) {
            const std::uint64_t y = (mt_[i] & kMtUM) | (mt_[(i + 1) % kMtN] & kMtLM);
            mt_[i] = mt_[(i + kMtM) % kMtN] ^ (y >> 1) ^ ((y & 1) ? kMtA : 0ull);
        }
        idx_ = 0;
    }
    std::uint64_t mt_[kMtN];
    int idx_ = kMtN;
};

// window 2^log2j words ahead (kMtJumpMinLog2 <= log2j <= kMtJumpMaxLog2)
inline void mt64_jump_pow2(const std::uint64_t* win, int log2j, std::uint64_t* out) {
    const unsigned long long* g = kMtJump[log2j - kMtJumpMinLog2];
    // x[0 .. 312 + 19937): the recurrence continued from the window
    std::vector<std::uint64_t> xs(kMtN + kMtDeg);
    std::memcpy(xs.data(), win, sizeof(std::uint64_t) * kMtN);
    for (int i = 0; i < kMtDeg; ++i) {
        const std::uint64_t y = (xs[i] & kMtUM) | (xs[i + 1] & kMtLM);
        xs[i + kMtN] = xs[i + kMtM] ^ (y >> 1) ^ ((y & 1) ? kMtA : 0ull);
    }
    std::uint64_t acc[kMtN] = {};
    for (int w = 0; w < kMtN; ++w) {
        unsigned long long bits = g[w];
        while (bits) {
            const int i = 64 * w + __builtin_ctzll(bits);
            bits &= bits - 1;
            const std::uint64_t* src = xs.data() + i;
            for (int t = 0; t < kMtN; ++t) acc[t] ^= src[t];
        }
    }
    std::memcpy(out, acc, sizeof(acc));
}

// window `words` ahead, words a multiple of 2^kMtJumpMinLog2 (binary decomposition)
inline bool mt64_jump(const std::uint64_t* win, std::uint64_t words, std::uint64_t* out) {
    if (words & ((1ull << kMtJumpMinLog2) - 1)) return false;
    if (kMtJumpMaxLog2 < 63 && (words >> (kMtJumpMaxLog2 + 1))) return false;
    std::uint64_t cur[kMtN];
    std::memcpy(cur, win, sizeof(cur));
    for (int j = kMtJumpMinLog2; j <= kMtJumpMaxLog2; ++j)
        if ((words >> j) & 1) {
            std::uint64_t nxt[kMtN];
            mt64_jump_pow2(cur, j, nxt);
            std::memcpy(cur, nxt, sizeof(cur));
        }
    std::memcpy(out, cur, sizeof(cur));
    return true;
}

}  // namespace nlsp_host
