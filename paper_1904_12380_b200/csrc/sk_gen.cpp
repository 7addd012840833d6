// sk_gen.cpp -- deterministic host-side input generators (include/softmax_b200.h).
//
// fill_uniform mirrors the reference generator (tensor.py:106-121): numpy's
// Philox4x64-10 raw stream keyed by `seed` (np.random.Philox(key=seed)), each
// raw u64 -> ((u >> 11) + 0.5) * 2^-53 -> low + (high-low)u in double -> float
// -> clamp into the open interval.  numpy increments the 256-bit counter before
// each 4-word block, so raw draw i comes from block i/4 with counter i/4 + 1.
// The normal generator and the sentinel planter are this framework's own
// definitions for the BASELINE configs (the reference has no normal generator).
#include <cmath>
#include <cstdint>
#include <thread>
#include <unordered_set>
#include <vector>

#include "../../include/softmax_b200.h"

namespace {

inline void mulhilo(uint64_t a, uint64_t b, uint64_t& hi, uint64_t& lo) {
  const __uint128_t p = static_cast<__uint128_t>(a) * b;
  hi = static_cast<uint64_t>(p >> 64);
  lo = static_cast<uint64_t>(p);
}

// Philox4x64-10 block `blk` (0-based) of the stream keyed by {seed, 0}.
inline void philox_block(uint64_t blk, uint64_t seed, uint64_t out[4]) {
  uint64_t c0 = blk + 1, c1 = (blk + 1 == 0) ? 1 : 0, c2 = 0, c3 = 0;
  uint64_t k0 = seed, k1 = 0;
  for (int r = 0; r < 10; ++r) {
    uint64_t hi0, lo0, hi1, lo1;
    mulhilo(0xD2E7470EE14C6C93ULL, c0, hi0, lo0);
    mulhilo(0xCA5A826395121157ULL, c2, hi1, lo1);
    const uint64_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
    k0 += 0x9E3779B97F4A7C15ULL;
    k1 += 0xBB67AE8584CAA73BULL;
  }
  out[0] = c0;
  out[1] = c1;
  out[2] = c2;
  out[3] = c3;
}

struct RawStream {  // sequential reader of raw draws from position `pos`
  uint64_t seed, pos;
  uint64_t buf[4];
  bool have = false;
  RawStream(uint64_t s, uint64_t p) : seed(s), pos(p) {}
  uint64_t next() {
    if (!have || (pos & 3) == 0) {
      philox_block(pos >> 2, seed, buf);
      have = true;
    }
    return buf[pos++ & 3];
  }
};

inline double open_unit(uint64_t u) {  // tensor.py:113
  return (static_cast<double>(u >> 11) + 0.5) * 0x1.0p-53;
}

template <class F>
void parallel_for(int64_t n, int nthreads, F&& f) {
  if (nthreads <= 0) nthreads = static_cast<int>(std::thread::hardware_concurrency());
  if (nthreads < 1) nthreads = 1;
  const int64_t min_per = 1 << 16;
  int64_t nt = std::min<int64_t>(nthreads, (n + min_per - 1) / min_per);
  if (nt <= 1) {
    f(int64_t(0), n);
    return;
  }
  // chunk boundaries on multiples of 4 keep Philox blocks whole per thread
  const int64_t per = ((n + nt - 1) / nt + 3) / 4 * 4;
  std::vector<std::thread> ts;
  for (int64_t t = 0; t < nt; ++t) {
    const int64_t a = t * per, b = std::min(n, a + per);
    if (a >= b) break;
    ts.emplace_back([&f, a, b] { f(a, b); });
  }
  for (auto& t : ts) t.join();
}

}  // namespace

extern "C" {

int sk_fill_uniform_f32(float* dst, int64_t n, uint64_t seed, double low, double high,
                        uint64_t start, int nthreads) {
  if (n < 0 || (n > 0 && !dst)) return SK_ERR_ARGUMENT;
  if (!std::isfinite(low) || !std::isfinite(high) || !(low < high)) return SK_ERR_ARGUMENT;
  const float lo = static_cast<float>(low), hi = static_cast<float>(high);
  // tensor.py:117-120: clamp into the open interval
  const float lo_in = (lo <= low) ? std::nextafter(lo, hi) : lo;
  const float hi_in = (hi >= high) ? std::nextafter(hi, lo) : hi;
  parallel_for(n, nthreads, [&](int64_t a, int64_t b) {
    RawStream rs(seed, start + static_cast<uint64_t>(a));
    for (int64_t i = a; i < b; ++i) {
      const double u = open_unit(rs.next());
      float v = static_cast<float>(low + (high - low) * u);
      v = v < lo_in ? lo_in : (v > hi_in ? hi_in : v);
      dst[i] = v;
    }
  });
  return SK_OK;
}

int sk_fill_normal_f32(float* dst, int64_t n, uint64_t seed, double sigma, uint64_t start,
                       int nthreads) {
  if (n < 0 || (n > 0 && !dst) || !(sigma > 0) || !std::isfinite(sigma)) return SK_ERR_ARGUMENT;
  const double two_pi = 6.283185307179586476925286766559;
  parallel_for(n, nthreads, [&](int64_t a, int64_t b) {
    // element i uses the pair (2*(i/2), 2*(i/2)+1) of raw draws (absolute index)
    for (int64_t i = a; i < b;) {
      const uint64_t gi = start + static_cast<uint64_t>(i);
      const uint64_t pair = gi >> 1;
      RawStream rs(seed, 2 * pair);
      const double u1 = open_unit(rs.next());
      const double u2 = open_unit(rs.next());
      const double rad = std::sqrt(-2.0 * std::log(u1));
      const double th = two_pi * u2;
      if ((gi & 1) == 0) {
        dst[i] = static_cast<float>(sigma * (rad * std::cos(th)));
        ++i;
        if (i < b) {
          dst[i] = static_cast<float>(sigma * (rad * std::sin(th)));
          ++i;
        }
      } else {
        dst[i] = static_cast<float>(sigma * (rad * std::sin(th)));
        ++i;
      }
    }
  });
  return SK_OK;
}

int sk_plant_f32(float* x, int64_t total, int64_t count, uint64_t seed, float value) {
  if (total < 0 || count < 0 || count > total || (total > 0 && !x)) return SK_ERR_ARGUMENT;
  RawStream rs(seed ^ 0x5EEDC0FFEEULL, 0);
  std::vector<uint8_t> seen(static_cast<size_t>(total), 0);
  int64_t placed = 0;
  while (placed < count) {
    const uint64_t idx = rs.next() % static_cast<uint64_t>(total);
    if (!seen[idx]) {
      seen[idx] = 1;
      x[idx] = value;
      ++placed;
    }
  }
  return SK_OK;
}

}  // extern "C"
