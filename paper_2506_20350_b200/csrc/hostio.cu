// Host-side helpers of the problem-file path (TBZ1, problems.py:219-322 of the reference).
#include "common.cuh"

extern "C" int toep_fnv1a64(const void* data, uint64_t bytes, uint64_t* out) {
  TOEP_REQUIRE(out != nullptr && (data != nullptr || bytes == 0), TOEP_ERR_ARG, "bad fnv1a64 arguments");
  const unsigned char* p = static_cast<const unsigned char*>(data);
  uint64_t h = 0xCBF29CE484222325ull;  // offset basis
  for (uint64_t i = 0; i < bytes; ++i) {
    h ^= p[i];
    h *= 0x100000001B3ull;  // FNV prime (wraps mod 2^64)
  }
  *out = h;
  return TOEP_OK;
}
