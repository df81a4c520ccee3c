// Test-only helper: the CUDA toolkit's HOST fp8 conversion (cuda_fp8.hpp,
// __nv_cvt_float_to_fp8 with __NV_SATFINITE) used as an independent library
// pin for oracle/fp8.py's encode.  Never linked
// into the product.  Usage:
//   fp8_host_cast e4m3|e5m2 <in.f32> <out.u8>      convert a file of float32
//   fp8_host_cast sweep e4m3|e5m2 <out.u8>          all 2^32 float32 bit patterns (NaN -> 0xFF marker)
#include <cuda_fp8.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cstdint>
#include <vector>

static __nv_fp8_interpretation_t interp(const char* s) {
  return std::strcmp(s, "e5m2") == 0 ? __NV_E5M2 : __NV_E4M3;
}

int main(int argc, char** argv) {
  if (argc == 4 && std::strcmp(argv[1], "sweep") != 0) {
    FILE* fi = std::fopen(argv[2], "rb");
    FILE* fo = std::fopen(argv[3], "wb");
    if (!fi || !fo) return 2;
    std::vector<float> buf(1 << 20);
    std::vector<unsigned char> ob(1 << 20);
    size_t n;
    while ((n = std::fread(buf.data(), 4, buf.size(), fi)) > 0) {
      for (size_t i = 0; i < n; ++i)
        ob[i] = (unsigned char)__nv_cvt_float_to_fp8(buf[i], __NV_SATFINITE, interp(argv[1]));
      std::fwrite(ob.data(), 1, n, fo);
    }
    std::fclose(fi); std::fclose(fo);
    return 0;
  }
  if (argc == 4) {  // sweep
    FILE* fo = std::fopen(argv[3], "wb");
    if (!fo) return 2;
    std::vector<unsigned char> ob(1u << 24);
    for (uint64_t base = 0; base < (1ull << 32); base += ob.size()) {
      for (uint32_t i = 0; i < ob.size(); ++i) {
        uint32_t bits = (uint32_t)(base + i);
        float f; std::memcpy(&f, &bits, 4);
        ob[i] = (unsigned char)__nv_cvt_float_to_fp8(f, __NV_SATFINITE, interp(argv[2]));
      }
      std::fwrite(ob.data(), 1, ob.size(), fo);
    }
    std::fclose(fo);
    return 0;
  }
  std::fprintf(stderr, "usage\n");
  return 1;
}
