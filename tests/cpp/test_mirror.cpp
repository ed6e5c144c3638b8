// C++ host-mirror test (include/specattn_b200.hpp): reference-shaped calls, reference exception types.
//   mode "cpu": host-only checks (no device call reaches the GPU)
//   mode "gpu": KvStore append / truncate / gather round trip on the device
#include <cmath>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <vector>

#include "specattn_b200.hpp"

using namespace specattn_b200;

#define EXPECT(cond)                                                  \
  do {                                                                \
    if (!(cond)) {                                                    \
      std::fprintf(stderr, "FAILED %s:%d %s\n", __FILE__, __LINE__, #cond); \
      return 1;                                                       \
    }                                                                 \
  } while (0)

template <typename E, typename F>
static bool throws(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

int main(int argc, char** argv) {
  const bool gpu = argc > 1 && std::strcmp(argv[1], "gpu") == 0;
  // selection_k KATs (selection.cpp:63-66): llround, clamp to [k_min, p]
  EXPECT(selection_k(0.07, 32768, 16) == 2294);
  EXPECT(selection_k(0.07, 131072, 16) == 9175);
  EXPECT(selection_k(0.25, 10, 16) == 10);
  EXPECT(selection_k(0.5, 5, 0) == 3);  // llround(2.5) = 3
  // invalid configuration -> std::invalid_argument before any device work
  ModelConfig bad;
  bad.n_layers = 0;  // ModelConfig::validate-style rejection
  EXPECT(throws<std::invalid_argument>([&] { KvStore kv(bad); }));
  ModelConfig bad_d;
  bad_d.head_dim = 64;  // not supported by the kernels (SA_NOT_SUPPORTED -> runtime_error)
  EXPECT(throws<std::runtime_error>([&] { KvStore kv(bad_d); }));
  ModelConfig badp;
  badp.page_size = 100;
  EXPECT(throws<std::invalid_argument>([&] { KvStore kv(badp); }));
  if (!gpu) {
    std::printf("mirror cpu ok\n");
    return 0;
  }
  ModelConfig cfg;
  cfg.n_layers = 2;
  cfg.n_kv_heads = 2;
  cfg.max_context = 300;
  cfg.page_size = 128;
  KvStore kv(cfg);
  EXPECT(kv.bytes_per_token() == 2 * 2 * 2 * 128 * 4);
  const int rows = 4;  // n_layers * n_kv_heads
  std::vector<float> k(rows * 128), v(rows * 128);
  for (int t = 0; t < 5; ++t) {
    for (int i = 0; i < rows * 128; ++i) {
      k[i] = static_cast<float>(t * 1000 + i) * 0.25f;  // bf16-representable
      v[i] = -k[i];
      k[i] = static_cast<float>(static_cast<int>(k[i]) % 256);
      v[i] = static_cast<float>(static_cast<int>(v[i]) % 256);
    }
    EXPECT(kv.append(k.data(), v.data()) == t + 1);
  }
  kv.truncate(3);  // 5 appends, truncate 3, append 1 -> len 4
  EXPECT(kv.size() == 3);
  EXPECT(kv.append(k.data(), v.data()) == 4);
  EXPECT(throws<std::out_of_range>([&] { kv.truncate(5); }));
  EXPECT(throws<std::out_of_range>([&] { kv.gather(1, 1, {2, 1}); }));  // not strictly increasing
  auto kvp = kv.gather(1, 1, {3});
  // token 3 = the last appended (t = 4 values), row layer 1 head 1 = row 3
  for (int c = 0; c < 128; ++c) EXPECT(kvp.first[c] == k[3 * 128 + c] && kvp.second[c] == v[3 * 128 + c]);
  std::vector<float> big(rows * 128, 0.f);
  while (kv.size() < cfg.max_context) kv.append(big.data(), big.data());
  EXPECT(throws<std::length_error>([&] { kv.append(big.data(), big.data()); }));
  std::printf("mirror gpu ok\n");
  return 0;
}
