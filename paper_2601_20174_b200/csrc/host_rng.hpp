// paper_2601_20174_b200/csrc/host_rng.hpp — restatement of the reference's
// random streams (rng.hpp:12-73) for host-side input generation: splitmix64
// mix_seed, std::mt19937_64, top-53-bit uniforms and Box–Muller with the cached
// sine value. normal_stream() is bit-identical to a serial loop over
// Rng(seed).normal(), produced by several threads that each jump their own
// generator to their slice of the one mt19937_64 stream (mt_jump.hpp).
#pragma once

#include <algorithm>
#include <array>
#include <atomic>
#include <cmath>
#include <condition_variable>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <random>
#include <thread>
#include <vector>

#include "mt_jump.hpp"

namespace nlsp_host {

inline std::uint64_t mix_seed(std::uint64_t seed, std::uint64_t tag) {
    std::uint64_t z = seed + 0x9e3779b97f4a7c15ULL * (tag + 1);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

class Rng {
public:
    explicit Rng(std::uint64_t seed) : gen_(seed) {}
    std::uint64_t u64() { return gen_(); }
    double uniform() { return static_cast<double>(gen_() >> 11) * 0x1.0p-53; }
    double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
    double normal() {
        if (has_cached_) {
            has_cached_ = false;
            return cached_;
        }
        double u1 = uniform();
        double u2 = uniform();
        while (u1 <= 0.0) u1 = uniform();
        const double r = std::sqrt(-2.0 * std::log(u1));
        const double a = 2.0 * 3.141592653589793 * u2;
        cached_ = r * std::sin(a);
        has_cached_ = true;
        return r * std::cos(a);
    }

private:
    std::mt19937_64 gen_;
    double cached_ = 0.0;
    bool has_cached_ = false;
};

// One Box-Muller pair of Rng::normal() (rng.hpp:37-49) from the uniforms u1, u2
inline void box_muller(double u1, double u2, double* c, double* s) {
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double a = 2.0 * 3.141592653589793 * u2;
    *c = r * std::cos(a);
    *s = r * std::sin(a);
}

// Serial continuation of the normal stream from a generator: pairs [base,
// pairs_total), chunk by chunk (the rejection loop `while (u1 <= 0) u1 =
// uniform()` of rng.hpp:43 consumes extra words, which only a sequential pass
// can follow).
template <class Sink>
inline void normal_stream_serial(Mt64& gen, std::uint64_t count, std::uint64_t base, Sink& sink,
                                 std::uint64_t chunk, double zero_below) {
    const std::uint64_t pairs_total = (count + 1) / 2;
    auto uni = [&]() { return static_cast<double>(gen() >> 11) * 0x1.0p-53; };
    while (base < pairs_total) {
        const std::uint64_t np = std::min(chunk, pairs_total - base);
        double* out = sink.buffer(base, np);
        for (std::uint64_t p = 0; p < np; ++p) {
            double u1 = uni();
            const double u2 = uni();
            while (u1 <= zero_below) u1 = uni();
            double c, s;
            box_muller(u1, u2, &c, &s);
            out[2 * p] = c;
            if (2 * (base + p) + 1 < count) out[2 * p + 1] = s;
        }
        sink.done(base, np);
        base += np;
    }
}

// The normal stream of Rng(seed).normal() x count, produced chunk by chunk:
// sink.buffer(base, np) gives the destination of pairs [base, base + np) (2 np
// doubles, the last one dropped when count is odd and the chunk is last), and
// sink.done(base, np) is called once they are written — in order, from this
// thread — so a caller can ship each chunk (e.g. to the device) while the
// next one is generated.
//
// Every output bit is that of a serial loop over Rng(seed).normal(), but the
// loop is not serial: pair p takes words 2p and 2p + 1 of the mt19937_64
// stream, so W worker threads each own one contiguous piece of every chunk and
// position their own generator there by jump-ahead (mt_jump.hpp) — once by
// w * piece words, then by one chunk per chunk. The draw and the Box-Muller
// transform both run on all threads. The one data-dependent step, the
// rejection of u1 = 0 (probability 2^-53 per pair), shifts the rest of the
// stream by a word: a worker that meets it raises a flag, the chunk is
// discarded and the stream continues serially from that chunk's start.
// zero_below (0 in production) widens the rejection for tests of that path.
template <class Sink>
inline void normal_stream_chunks(std::uint64_t seed, std::uint64_t count, Sink& sink,
                                 std::uint64_t chunk = 1ull << 22, double zero_below = 0.0,
                                 unsigned max_workers = 0) {
    const std::uint64_t pairs_total = (count + 1) / 2;
    if (pairs_total == 0) return;
    std::uint64_t win0[kMtN];
    mt64_seed(seed, win0);
    // workers: a power of two, every piece a power of two of at least 2^16 pairs
    // (= 2^17 words, the smallest tabulated jump)
    unsigned hw = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
    if (max_workers) hw = std::min(hw, max_workers);
    unsigned W = 1;
    const bool pow2 = (chunk & (chunk - 1)) == 0;
    while (pow2 && 2 * W <= hw && chunk / (2 * W) >= (1ull << (kMtJumpMinLog2 - 1))) W *= 2;
    if (W == 1 || pairs_total < chunk) {
        Mt64 gen(win0);
        normal_stream_serial(gen, count, 0, sink, chunk, zero_below);
        return;
    }
    const std::uint64_t piece = chunk / W;  // pairs per worker and chunk
    struct Shared {
        std::mutex mu;
        std::condition_variable cv_go, cv_done;
        std::uint64_t epoch = 0;  // chunk generation counter
        unsigned pending = 0;
        bool quit = false;
        double* out = nullptr;
        std::uint64_t base = 0, np = 0;
        std::atomic<bool> zero{false};
    } sh;
    std::vector<std::array<std::uint64_t, kMtN>> start(W);  // each worker's window at its piece of the current chunk
    auto worker = [&](unsigned w) {
        // position: w pieces into the stream (2 words per pair)
        std::uint64_t cur[kMtN];
        mt64_jump(win0, 2 * piece * w, cur);
        std::memcpy(start[w].data(), cur, sizeof(cur));
        std::uint64_t seen = 0;
        for (;;) {
            double* out;
            std::uint64_t base, np;
            {
                std::unique_lock<std::mutex> lk(sh.mu);
                sh.cv_go.wait(lk, [&] { return sh.quit || sh.epoch != seen; });
                if (sh.quit) return;
                seen = sh.epoch;
                out = sh.out;
                base = sh.base;
                np = sh.np;
            }
            const std::uint64_t lo = std::min(np, piece * w), hi = std::min(np, lo + piece);
            Mt64 gen(start[w].data());
            for (std::uint64_t p = lo; p < hi; ++p) {
                const double u1 = static_cast<double>(gen() >> 11) * 0x1.0p-53;
                const double u2 = static_cast<double>(gen() >> 11) * 0x1.0p-53;
                if (u1 <= zero_below) {
                    sh.zero.store(true, std::memory_order_relaxed);
                    break;
                }
                double c, s;
                box_muller(u1, u2, &c, &s);
                out[2 * p] = c;
                if (2 * (base + p) + 1 < count) out[2 * p + 1] = s;
            }
            // next chunk's start: one chunk of words ahead of this one's
            if (base + np < pairs_total) {
                std::uint64_t nxt[kMtN];
                mt64_jump(start[w].data(), 2 * chunk, nxt);
                std::memcpy(cur, nxt, sizeof(cur));
            }
            {
                std::lock_guard<std::mutex> lk(sh.mu);
                // published after the chunk so a fallback still finds this chunk's start
                std::memcpy(start[w].data(), cur, sizeof(cur));
                if (--sh.pending == 0) sh.cv_done.notify_one();
            }
        }
    };
    std::vector<std::thread> th;
    for (unsigned w = 0; w < W; ++w) th.emplace_back(worker, w);
    auto stop = [&] {
        {
            std::lock_guard<std::mutex> lk(sh.mu);
            sh.quit = true;
        }
        sh.cv_go.notify_all();
        for (auto& t : th) t.join();
    };
    std::uint64_t chunk_win[kMtN];  // the stream's window at the current chunk's start
    std::memcpy(chunk_win, win0, sizeof(chunk_win));
    for (std::uint64_t base = 0; base < pairs_total;) {
        const std::uint64_t np = std::min(chunk, pairs_total - base);
        double* out = sink.buffer(base, np);
        {
            std::lock_guard<std::mutex> lk(sh.mu);
            sh.out = out;
            sh.base = base;
            sh.np = np;
            sh.pending = W;
            ++sh.epoch;
        }
        sh.cv_go.notify_all();
        // this thread: the next chunk's start window, for the serial fallback
        std::uint64_t next_win[kMtN];
        if (base + np < pairs_total) mt64_jump(chunk_win, 2 * chunk, next_win);
        {
            std::unique_lock<std::mutex> lk(sh.mu);
            sh.cv_done.wait(lk, [&] { return sh.pending == 0; });
        }
        if (sh.zero.load()) {
            // a rejected u1 in this chunk: redo it and the rest serially
            stop();
            Mt64 gen(chunk_win);
            struct Redo {  // the first chunk's buffer is already held
                Sink& s;
                double* held;
                double* buffer(std::uint64_t b, std::uint64_t n) {
                    if (held) {
                        double* h = held;
                        held = nullptr;
                        return h;
                    }
                    return s.buffer(b, n);
                }
                void done(std::uint64_t b, std::uint64_t n) { s.done(b, n); }
            } redo{sink, out};
            normal_stream_serial(gen, count, base, redo, chunk, zero_below);
            return;
        }
        sink.done(base, np);
        base += np;
        std::memcpy(chunk_win, next_win, sizeof(chunk_win));
    }
    stop();
}

// the whole stream into out (count doubles)
inline void normal_stream(std::uint64_t seed, std::uint64_t count, double* out) {
    struct ToArray {
        double* out;
        std::uint64_t count;
        std::vector<double> scratch;  // an odd count's last pair: one value past the end
        double* buffer(std::uint64_t base, std::uint64_t np) {
            if (2 * (base + np) <= count) return out + 2 * base;
            scratch.assign(2 * np, 0.0);
            return scratch.data();
        }
        void done(std::uint64_t base, std::uint64_t np) {
            if (2 * (base + np) > count)
                std::copy(scratch.begin(), scratch.begin() + (count - 2 * base), out + 2 * base);
        }
    } sink{out, count, {}};
    normal_stream_chunks(seed, count, sink);
}

// S^(0) of generate_smoothed_vectors before the sweeps (smoothing.hpp:84-92)
inline void smoothed_s0(std::uint64_t seed, std::uint64_t n, std::uint64_t m,
                        const std::uint8_t* mask, double* out) {
    std::uint64_t live = 0;
    for (std::uint64_t i = 0; i < n; ++i) live += (mask && mask[i]) ? 0 : 1;
    const std::uint64_t s = mix_seed(seed, 0x736d6f6f);
    if (live == n) {
        normal_stream(s, n * m, out);
        return;
    }
    std::vector<double> tmp(live * m);
    normal_stream(s, tmp.size(), tmp.data());
    std::uint64_t k = 0;
    for (std::uint64_t i = 0; i < n; ++i) {
        double* row = out + i * m;
        if (mask && mask[i]) {
            std::fill(row, row + m, 0.0);
        } else {
            std::copy(tmp.begin() + k * m, tmp.begin() + (k + 1) * m, row);
            ++k;
        }
    }
}

}  // namespace nlsp_host
