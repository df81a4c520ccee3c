// Test-only helper: the CUDA toolkit's HOST fp4 conversion (cuda_fp4.hpp __nv_cvt_float_to_fp4
// with __NV_E2M1, cudaRoundNearest) used as an independent library pin for oracle/nvfp4.py's
// E2M1 encode (D35).  Never linked into the product.  Usage:
//   fp4_host_cast <in.f32> <out.u8>      convert a file of float32 (one code per byte)
//   fp4_host_cast sweep <out.u8>         all 2^32 float32 bit patterns (NaN inputs -> 0xFF)
#include <cuda_fp4.h>
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cmath>
#include <vector>

static unsigned char cvt(float f) {
  if (std::isnan(f)) return 0xFF;
  return (unsigned char)__nv_cvt_float_to_fp4(f, __NV_E2M1, cudaRoundNearest);
}

int main(int argc, char** argv) {
  if (argc == 3 && std::strcmp(argv[1], "sweep") != 0) {
    FILE* fi = std::fopen(argv[1], "rb");
    FILE* fo = std::fopen(argv[2], "wb");
    if (!fi || !fo) return 2;
    std::vector<float> buf(1 << 20);
    std::vector<unsigned char> ob(1 << 20);
    size_t n;
    while ((n = std::fread(buf.data(), 4, buf.size(), fi)) > 0) {
      for (size_t i = 0; i < n; ++i) ob[i] = cvt(buf[i]);
      std::fwrite(ob.data(), 1, n, fo);
    }
    std::fclose(fi);
    std::fclose(fo);
    return 0;
  }
  if (argc == 3) {
    FILE* fo = std::fopen(argv[2], "wb");
    if (!fo) return 2;
    std::vector<unsigned char> ob(1u << 24);
    for (uint64_t base = 0; base < (1ull << 32); base += ob.size()) {
      for (uint32_t i = 0; i < ob.size(); ++i) {
        const uint32_t bits = (uint32_t)(base + i);
        float f;
        std::memcpy(&f, &bits, 4);
        ob[i] = cvt(f);
      }
      std::fwrite(ob.data(), 1, ob.size(), fo);
    }
    std::fclose(fo);
    return 0;
  }
  std::fprintf(stderr, "usage\n");
  return 1;
}
