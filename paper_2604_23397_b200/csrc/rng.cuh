// Counter-based generators shared by host and device.
//
// philox4x64_10: Random123 Philox4x64 with 10 rounds, as used by numpy's
// `np.random.Philox` (the reference's `rng.stream`, rng.py:24-34).  numpy
// increments counter word 0 before generating, so the first 64-bit output of
// stream(seed, purpose, slot) is word 0 of philox(ctr={1, slot, 0, 0},
// key={seed, blake2b64(purpose)}), and Generator.random() maps it to
// (u >> 11) * 2^-53.
//
// blake2b64: BLAKE2b (RFC 7693) with an 8-byte digest, unkeyed, for messages
// of at most 128 bytes (one compression) -- `hashlib.blake2b(..., digest_size=8)`
// read little-endian, as in rng.py:17-21 and phy_pipeline.py:347-350.
#pragma once
#include <stdint.h>

#ifdef __CUDACC__
#define ARCHES_HD __host__ __device__ __forceinline__
#else
#define ARCHES_HD inline
#endif

namespace arches_rng {

ARCHES_HD uint64_t mulhi64(uint64_t a, uint64_t b) {
#ifdef __CUDA_ARCH__
  return __umul64hi(a, b);
#else
  return (uint64_t)(((unsigned __int128)a * b) >> 64);
#endif
}

ARCHES_HD void philox4x64_10(uint64_t ctr[4], uint64_t k0, uint64_t k1) {
  const uint64_t M0 = 0xD2E7470EE14C6C93ull, M1 = 0xCA5A826395121157ull;
  const uint64_t W0 = 0x9E3779B97F4A7C15ull, W1 = 0xBB67AE8584CAA73Bull;
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += W0;
      k1 += W1;
    }
    const uint64_t hi0 = mulhi64(M0, ctr[0]), lo0 = M0 * ctr[0];
    const uint64_t hi1 = mulhi64(M1, ctr[2]), lo1 = M1 * ctr[2];
    const uint64_t c1 = ctr[1], c3 = ctr[3];
    ctr[0] = hi1 ^ c1 ^ k0;
    ctr[1] = lo1;
    ctr[2] = hi0 ^ c3 ^ k1;
    ctr[3] = lo0;
  }
}

// first Generator.random() double of stream(seed, purpose, slot)
ARCHES_HD double stream_first_uniform(uint64_t seed, uint64_t purpose_key, uint64_t slot) {
  uint64_t c[4] = {1ull, slot, 0ull, 0ull};
  philox4x64_10(c, seed, purpose_key);
  return (double)(c[0] >> 11) * (1.0 / 9007199254740992.0);
}

// Generator.random() double number `idx` (0-based) of stream(seed, purpose, slot):
// numpy's Philox buffers four outputs per counter, counter word 0 pre-incremented
ARCHES_HD double stream_uniform_at(uint64_t seed, uint64_t purpose_key, uint64_t slot,
                                   uint64_t idx) {
  uint64_t c[4] = {1ull + (idx >> 2), slot, 0ull, 0ull};
  philox4x64_10(c, seed, purpose_key);
  return (double)(c[idx & 3] >> 11) * (1.0 / 9007199254740992.0);
}

#ifdef __CUDACC__
// element e of complex_normal(stream(seed, purpose, slot), shape) with n elements
// (rng.py:37-47): u1 = random #e, u2 = random #(n + e), sqrt(-log1p(-u1)) *
// (cos, sin)(2 pi u2) -- numpy's operation order; libm-level (<= 2 ulp) rounding
__device__ __forceinline__ double2 complex_normal_at(uint64_t seed, uint64_t purpose_key,
                                                     uint64_t slot, uint64_t n, uint64_t e) {
  const double u1 = stream_uniform_at(seed, purpose_key, slot, e);
  const double u2 = stream_uniform_at(seed, purpose_key, slot, n + e);
  const double r = sqrt(-log1p(-u1));
  const double th = 6.283185307179586 * u2;  // (2j * np.pi) * u2: imaginary part
  double sn, cs;
  sincos(th, &sn, &cs);
  return make_double2(r * cs, r * sn);
}
#endif

ARCHES_HD uint64_t rotr64(uint64_t x, int n) { return (x >> n) | (x << (64 - n)); }

ARCHES_HD void b2_g(uint64_t* v, int a, int b, int c, int d, uint64_t x, uint64_t y) {
  v[a] = v[a] + v[b] + x;
  v[d] = rotr64(v[d] ^ v[a], 32);
  v[c] = v[c] + v[d];
  v[b] = rotr64(v[b] ^ v[c], 24);
  v[a] = v[a] + v[b] + y;
  v[d] = rotr64(v[d] ^ v[a], 16);
  v[c] = v[c] + v[d];
  v[b] = rotr64(v[b] ^ v[c], 63);
}

// BLAKE2b-64 of len <= 128 bytes
ARCHES_HD uint64_t blake2b64(const uint8_t* msg, int len) {
  const uint64_t iv[8] = {0x6a09e667f3bcc908ull, 0xbb67ae8584caa73bull, 0x3c6ef372fe94f82bull,
                          0xa54ff53a5f1d36f1ull, 0x510e527fade682d1ull, 0x9b05688c2b3e6c1full,
                          0x1f83d9abfb41bd6bull, 0x5be0cd19137e2179ull};
  const uint8_t sigma[12][16] = {
      {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15},
      {14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3},
      {11, 8, 12, 0, 5, 2, 15, 13, 10, 14, 3, 6, 7, 1, 9, 4},
      {7, 9, 3, 1, 13, 12, 11, 14, 2, 6, 5, 10, 4, 0, 15, 8},
      {9, 0, 5, 7, 2, 4, 10, 15, 14, 1, 11, 12, 6, 8, 3, 13},
      {2, 12, 6, 10, 0, 11, 8, 3, 4, 13, 7, 5, 15, 14, 1, 9},
      {12, 5, 1, 15, 14, 13, 4, 10, 0, 7, 6, 3, 9, 2, 8, 11},
      {13, 11, 7, 14, 12, 1, 3, 9, 5, 0, 15, 4, 8, 6, 2, 10},
      {6, 15, 14, 9, 11, 3, 0, 8, 12, 2, 13, 7, 1, 4, 10, 5},
      {10, 2, 8, 4, 7, 6, 1, 5, 15, 11, 9, 14, 3, 12, 13, 0},
      {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15},
      {14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3}};
  uint64_t m[16];
  for (int i = 0; i < 16; ++i) m[i] = 0;
  for (int i = 0; i < len; ++i) m[i >> 3] |= (uint64_t)msg[i] << (8 * (i & 7));
  uint64_t h0 = iv[0] ^ 0x01010008ull;  // digest 8, key 0, fanout 1, depth 1
  uint64_t v[16];
  v[0] = h0;
  for (int i = 1; i < 8; ++i) v[i] = iv[i];
  for (int i = 0; i < 8; ++i) v[8 + i] = iv[i];
  v[12] ^= (uint64_t)len;
  v[14] = ~v[14];  // final block
  for (int r = 0; r < 12; ++r) {
    const uint8_t* s = sigma[r];
    b2_g(v, 0, 4, 8, 12, m[s[0]], m[s[1]]);
    b2_g(v, 1, 5, 9, 13, m[s[2]], m[s[3]]);
    b2_g(v, 2, 6, 10, 14, m[s[4]], m[s[5]]);
    b2_g(v, 3, 7, 11, 15, m[s[6]], m[s[7]]);
    b2_g(v, 0, 5, 10, 15, m[s[8]], m[s[9]]);
    b2_g(v, 1, 6, 11, 12, m[s[10]], m[s[11]]);
    b2_g(v, 2, 7, 8, 13, m[s[12]], m[s[13]]);
    b2_g(v, 3, 4, 9, 14, m[s[14]], m[s[15]]);
  }
  return h0 ^ v[0] ^ v[8];
}

// BLAKE2b-64 of a message of len <= 32 bytes held in four little-endian words
// (register-only form: rounds unrolled, message schedule resolved at compile time)
#ifdef __CUDACC__
__device__ __forceinline__ uint64_t blake2b64_short(const uint64_t m0, const uint64_t m1,
                                                    const uint64_t m2, const uint64_t m3, int len) {
  constexpr uint8_t sg[12][16] = {
      {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15},
      {14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3},
      {11, 8, 12, 0, 5, 2, 15, 13, 10, 14, 3, 6, 7, 1, 9, 4},
      {7, 9, 3, 1, 13, 12, 11, 14, 2, 6, 5, 10, 4, 0, 15, 8},
      {9, 0, 5, 7, 2, 4, 10, 15, 14, 1, 11, 12, 6, 8, 3, 13},
      {2, 12, 6, 10, 0, 11, 8, 3, 4, 13, 7, 5, 15, 14, 1, 9},
      {12, 5, 1, 15, 14, 13, 4, 10, 0, 7, 6, 3, 9, 2, 8, 11},
      {13, 11, 7, 14, 12, 1, 3, 9, 5, 0, 15, 4, 8, 6, 2, 10},
      {6, 15, 14, 9, 11, 3, 0, 8, 12, 2, 13, 7, 1, 4, 10, 5},
      {10, 2, 8, 4, 7, 6, 1, 5, 15, 11, 9, 14, 3, 12, 13, 0},
      {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15},
      {14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3}};
  uint64_t m[16] = {m0, m1, m2, m3, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  const uint64_t h0 = 0x6a09e667f3bcc908ull ^ 0x01010008ull;
  uint64_t v[16] = {h0, 0xbb67ae8584caa73bull, 0x3c6ef372fe94f82bull, 0xa54ff53a5f1d36f1ull,
                    0x510e527fade682d1ull, 0x9b05688c2b3e6c1full, 0x1f83d9abfb41bd6bull,
                    0x5be0cd19137e2179ull, 0x6a09e667f3bcc908ull, 0xbb67ae8584caa73bull,
                    0x3c6ef372fe94f82bull, 0xa54ff53a5f1d36f1ull, 0x510e527fade682d1ull,
                    0x9b05688c2b3e6c1full, 0x1f83d9abfb41bd6bull, 0x5be0cd19137e2179ull};
  v[12] ^= (uint64_t)len;
  v[14] = ~v[14];
#pragma unroll
  for (int r = 0; r < 12; ++r) {
    b2_g(v, 0, 4, 8, 12, m[sg[r][0]], m[sg[r][1]]);
    b2_g(v, 1, 5, 9, 13, m[sg[r][2]], m[sg[r][3]]);
    b2_g(v, 2, 6, 10, 14, m[sg[r][4]], m[sg[r][5]]);
    b2_g(v, 3, 7, 11, 15, m[sg[r][6]], m[sg[r][7]]);
    b2_g(v, 0, 5, 10, 15, m[sg[r][8]], m[sg[r][9]]);
    b2_g(v, 1, 6, 11, 12, m[sg[r][10]], m[sg[r][11]]);
    b2_g(v, 2, 7, 8, 13, m[sg[r][12]], m[sg[r][13]]);
    b2_g(v, 3, 4, 9, 14, m[sg[r][14]], m[sg[r][15]]);
  }
  return h0 ^ v[0] ^ v[8];
}

// _lcid4_jitter(slot) without byte buffers: "lcid4:" + decimal digits packed
// straight into the message words
__device__ __forceinline__ double lcid4_jitter_fast(uint64_t slot) {
  int nd = 1;
  for (uint64_t t = slot / 10ull; t; t /= 10ull) ++nd;
  uint64_t w0 = 0x3a346469636cull, w1 = 0, w2 = 0, w3 = 0;  // "lcid4:" little-endian
  uint64_t x = slot;
#pragma unroll
  for (int k = 0; k < 20; ++k) {  // digit k from the right sits at byte 6 + nd - 1 - k
    if (k < nd) {
      const uint64_t dgt = x % 10ull;
      x /= 10ull;
      const int pos = 6 + nd - 1 - k;
      const uint64_t val = (uint64_t)('0' + (int)dgt) << (8 * (pos & 7));
      const int wd = pos >> 3;
      w0 |= wd == 0 ? val : 0ull;
      w1 |= wd == 1 ? val : 0ull;
      w2 |= wd == 2 ? val : 0ull;
      w3 |= wd == 3 ? val : 0ull;
    }
  }
  const uint64_t h = blake2b64_short(w0, w1, w2, w3, 6 + nd);
  const double xd = __ull2double_rn(h);
  return __dsub_rn(__dmul_rn(xd * (1.0 / 18446744073709551616.0), 2.0), 1.0);
}
#endif

// _lcid4_jitter(slot): blake2b64("lcid4:<slot>") / 2^64 * 2 - 1
ARCHES_HD double lcid4_jitter(uint64_t slot) {
#ifdef __CUDA_ARCH__
  return lcid4_jitter_fast(slot);
#endif
  uint8_t buf[32];
  const char* pre = "lcid4:";
  int n = 0;
  for (; n < 6; ++n) buf[n] = (uint8_t)pre[n];
  char dig[24];
  int nd = 0;
  do {
    dig[nd++] = (char)('0' + (int)(slot % 10ull));
    slot /= 10ull;
  } while (slot);
  while (nd) buf[n++] = (uint8_t)dig[--nd];
  const uint64_t h = blake2b64(buf, n);
#ifdef __CUDA_ARCH__
  const double x = __ull2double_rn(h);
  return __dsub_rn(__dmul_rn(x * (1.0 / 18446744073709551616.0), 2.0), 1.0);
#else
  volatile double x = (double)h;
  volatile double q = x / 18446744073709551616.0;
  volatile double t = q * 2.0;
  return t - 1.0;
#endif
}

}  // namespace arches_rng
