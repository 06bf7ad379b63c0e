// parsa/rng.hpp — host view of the counter-based chain streams.
//
// B200 drop-in for the reference header of the same name
// (/root/reference/proj/include/parsa/rng.hpp:1-95).  The bit contract is the
// reference's (rng.hpp:13-18, docs/rng.md:16-29):
//
//     draw i of stream (seed, chain, level)
//       = Philox4x32-10(counter {lo32 i, hi32 i, chain, level},
//                       key {lo32 seed, hi32 seed})
//     u = ((out1 << 32 | out0) >> 11) * 2^-53
//
// The device engines never touch this class: every chain regenerates its
// stream inside the kernel from (seed, chain, level) alone (csrc/philox.cuh).
// A host UniformStream exists because the reference API hands streams to the
// caller (ChainState, compute_neighbour, metropolis_accept); when such a
// stream is passed to parsa::metropolis_sweep its key and draw counter are
// shipped to the device, which continues it draw for draw.
#pragma once

#include <cstdint>

namespace parsa {

// Identity of one stream: the master seed plus the (chain, level) pair.
struct StreamKey {
    std::uint64_t master_seed = 0;
    std::uint32_t chain_index = 0;
    std::uint32_t level_index = 0;
};

namespace detail {

// Philox4x32 round multipliers and Weyl key increments (Salmon et al. SC'11).
inline constexpr std::uint32_t kPhiloxM0 = 0xD2511F53u;
inline constexpr std::uint32_t kPhiloxM1 = 0xCD9E8D57u;
inline constexpr std::uint32_t kPhiloxW0 = 0x9E3779B9u;
inline constexpr std::uint32_t kPhiloxW1 = 0xBB67AE85u;

struct Block4x32 {
    std::uint32_t v[4];
};

// Ten rounds of the Philox S-box network; the key is bumped after every
// round.  Same function as csrc/philox.cuh:philox4x32_10 (device copy).
inline Block4x32 philox4x32_10(Block4x32 x, std::uint32_t k0, std::uint32_t k1) {
    for (int r = 0; r < 10; ++r, k0 += kPhiloxW0, k1 += kPhiloxW1) {
        const std::uint64_t a = static_cast<std::uint64_t>(x.v[0]) * kPhiloxM0;
        const std::uint64_t b = static_cast<std::uint64_t>(x.v[2]) * kPhiloxM1;
        const std::uint32_t y0 = static_cast<std::uint32_t>(b >> 32) ^ x.v[1] ^ k0;
        const std::uint32_t y2 = static_cast<std::uint32_t>(a >> 32) ^ x.v[3] ^ k1;
        x.v[1] = static_cast<std::uint32_t>(b);
        x.v[3] = static_cast<std::uint32_t>(a);
        x.v[0] = y0;
        x.v[2] = y2;
    }
    return x;
}

} // namespace detail

class UniformStream {
public:
    UniformStream() = default;
    explicit UniformStream(StreamKey key) : key_(key) {}

    // Uniform in [0, 1) from draw number draws(); the counter moves by one.
    double next_uniform() {
        const std::uint64_t i = counter_++;
        const detail::Block4x32 out = detail::philox4x32_10(
            {{static_cast<std::uint32_t>(i), static_cast<std::uint32_t>(i >> 32), key_.chain_index,
              key_.level_index}},
            static_cast<std::uint32_t>(key_.master_seed),
            static_cast<std::uint32_t>(key_.master_seed >> 32));
        const std::uint64_t bits = static_cast<std::uint64_t>(out.v[1]) << 32 | out.v[0];
        return static_cast<double>(bits >> 11) * 0x1.0p-53;
    }

    // Coordinate index int(u * n) clamped to n - 1: exactly one draw.
    int next_coordinate_index(int n) {
        const int d = static_cast<int>(next_uniform() * static_cast<double>(n));
        return d < n ? d : n - 1;
    }

    // Draws consumed so far (the counter of the next draw).
    std::uint64_t draws() const { return counter_; }

    // B200 additions: what the device needs to continue this stream.
    const StreamKey& key() const { return key_; }
    void set_draws(std::uint64_t counter) { counter_ = counter; }

private:
    StreamKey key_{};
    std::uint64_t counter_ = 0;
};

inline UniformStream make_stream(StreamKey key) { return UniformStream(key); }

} // namespace parsa
