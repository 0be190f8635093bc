// Golden vectors for harness.format_double: std::to_chars(double) of libstdc++
// (the reference formats every CSV/JSON number this way, harness.cpp:199-203).
// g++ -std=c++17 -O2 gen_to_chars.cpp -o /tmp/g && /tmp/g > to_chars.txt
#include <charconv>
#include <cstdio>
#include <cstring>
#include <random>
#include <cmath>
int main() {
  std::mt19937_64 g(7);
  double fixed[] = {1e-06,0.001,0.0001,100000.0,123456.0,0.1,1.5,2.0,-3.25,1e22,5e-324,1200000.0,120.0,1e16,1.2345678901234568e+17,0.0,-0.0,1.7976931348623157e308,2.5e-07,31.41592653589793};
  char buf[64];
  for (double v : fixed) { auto r = std::to_chars(buf, buf+64, v); *r.ptr=0; printf("%.17g %s\n", v, buf); }
  for (int i = 0; i < 3000; ++i) {
    uint64_t b = g(); double v; std::memcpy(&v, &b, 8);
    if (!std::isfinite(v)) continue;
    if (i % 3 == 0) v = std::ldexp((double)(g() % 100000), (int)(g() % 80) - 40);
    auto r = std::to_chars(buf, buf+64, v); *r.ptr=0; printf("%a %s\n", v, buf);
  }
}
