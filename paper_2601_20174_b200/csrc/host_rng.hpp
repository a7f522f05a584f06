// paper_2601_20174_b200/csrc/host_rng.hpp — restatement of the reference's
// random streams (rng.hpp:12-73) for host-side input generation: splitmix64
// mix_seed, std::mt19937_64, top-53-bit uniforms and Box–Muller with the cached
// sine value. normal_stream() is bit-identical to a serial loop over
// Rng(seed).normal(); only the transcendental part runs on several threads.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <random>
#include <thread>
#include <vector>

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

// The normal stream of Rng(seed).normal() x count, produced chunk by chunk:
// sink.buffer(base, np) gives the destination of pairs [base, base + np) (2 np
// doubles, the last one dropped when count is odd and the chunk is last), and
// sink.done(base, np) is called once they are written — in order, from this
// thread — so a caller can ship each chunk (e.g. to the device) while the
// next one is generated.
template <class Sink>
inline void normal_stream_chunks(std::uint64_t seed, std::uint64_t count, Sink& sink,
                                 std::uint64_t chunk = 1ull << 22) {
    std::mt19937_64 gen(seed);
    auto uni = [&]() { return static_cast<double>(gen() >> 11) * 0x1.0p-53; };
    const std::uint64_t pairs_total = (count + 1) / 2;
    const std::uint64_t cap = std::min(chunk, pairs_total);
    // the sequential uniform stream of chunk c + 1 is drawn while the worker
    // threads run the Box-Muller transforms of chunk c (double-buffered); the
    // per-element arithmetic, and so every output bit, is that of a serial loop
    std::vector<double> u1[2] = {std::vector<double>(cap), std::vector<double>(cap)};
    std::vector<double> u2[2] = {std::vector<double>(cap), std::vector<double>(cap)};
    const unsigned hw = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
    auto draw = [&](std::uint64_t np, int buf) {
        for (std::uint64_t p = 0; p < np; ++p) {
            double a = uni();
            const double b = uni();
            while (a <= 0.0) a = uni();
            u1[buf][p] = a;
            u2[buf][p] = b;
        }
    };
    auto transform = [&](double* out, std::uint64_t base, int buf, std::uint64_t lo, std::uint64_t hi) {
        for (std::uint64_t p = lo; p < hi; ++p) {
            const double r = std::sqrt(-2.0 * std::log(u1[buf][p]));
            const double a = 2.0 * 3.141592653589793 * u2[buf][p];
            const std::uint64_t o = 2 * p;
            out[o] = r * std::cos(a);
            if (2 * (base + p) + 1 < count) out[o + 1] = r * std::sin(a);
        }
    };
    if (pairs_total == 0) return;
    std::uint64_t np = std::min(chunk, pairs_total);
    draw(np, 0);
    int buf = 0;
    for (std::uint64_t base = 0; base < pairs_total;) {
        const std::uint64_t next = base + np;
        const std::uint64_t np_next = next < pairs_total ? std::min(chunk, pairs_total - next) : 0;
        double* out = sink.buffer(base, np);
        if (np < 65536 || hw == 1) {
            transform(out, base, buf, 0, np);
            if (np_next) draw(np_next, buf ^ 1);
        } else {
            std::vector<std::thread> th;
            const unsigned workers = hw > 1 ? hw - 1 : 1;  // this thread draws the next chunk
            const std::uint64_t per = (np + workers - 1) / workers;
            for (unsigned t = 0; t < workers; ++t) {
                const std::uint64_t lo = t * per, hi = std::min(np, lo + per);
                if (lo < hi) th.emplace_back(transform, out, base, buf, lo, hi);
            }
            if (np_next) draw(np_next, buf ^ 1);
            for (auto& x : th) x.join();
        }
        sink.done(base, np);
        base = next;
        np = np_next;
        buf ^= 1;
    }
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
