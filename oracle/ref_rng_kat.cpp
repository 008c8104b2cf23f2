// Known-answer driver for the REFERENCE Rng: compiled against the reference's
// own header (/root/reference/proj/include/frag/common.hpp:45-100) by
// oracle/Makefile into oracle/_ref/rng_kat. Prints JSON golden vectors that
// oracle/gen_golden.py stores under tests/golden/rng_kat.json. Test
// infrastructure only.
#include <cstdio>

#include "frag/common.hpp"

int main() {
  const unsigned long long seeds[] = {0ULL, 1ULL, 7ULL, 42ULL, 1234ULL, 0xdeadbeefcafef00dULL};
  std::printf("{\n");
  bool first = true;
  for (unsigned long long s : seeds) {
    if (!first) std::printf(",\n");
    first = false;
    std::printf("  \"%llu\": {\n", s);
    {
      frag::Rng r(s);
      std::printf("    \"next_u64\": [");
      for (int i = 0; i < 16; ++i) std::printf("%s\"%llu\"", i ? ", " : "", (unsigned long long)r.next_u64());
      std::printf("],\n");
    }
    {
      frag::Rng r(s);
      std::printf("    \"normal\": [");
      for (int i = 0; i < 16; ++i) std::printf("%s%.17g", i ? ", " : "", r.normal());
      std::printf("],\n");
    }
    {
      frag::Rng r(s);
      std::printf("    \"normal_f_0.02\": [");
      for (int i = 0; i < 16; ++i) std::printf("%s%.9g", i ? ", " : "", (double)r.normal_f(0.02f));
      std::printf("],\n");
    }
    {
      frag::Rng r(s);
      std::printf("    \"below_256\": [");
      for (int i = 0; i < 32; ++i) std::printf("%s%llu", i ? ", " : "", (unsigned long long)r.below(256));
      std::printf("],\n");
    }
    {
      frag::Rng r(s);
      std::printf("    \"below_128256\": [");
      for (int i = 0; i < 32; ++i) std::printf("%s%llu", i ? ", " : "", (unsigned long long)r.below(128256));
      std::printf("],\n");
    }
    {
      frag::Rng r(s);
      std::printf("    \"next_float\": [");
      for (int i = 0; i < 16; ++i) std::printf("%s%.9g", i ? ", " : "", (double)r.next_float());
      std::printf("],\n");
    }
    {
      frag::Rng r(s);
      std::printf("    \"range_m5_5\": [");
      for (int i = 0; i < 16; ++i) std::printf("%s%lld", i ? ", " : "", (long long)r.range(-5, 5));
      std::printf("]\n");
    }
    std::printf("  }");
  }
  std::printf("\n}\n");
  return 0;
}
