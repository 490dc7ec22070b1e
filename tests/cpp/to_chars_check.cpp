// Prints std::to_chars(double) -- lpopt::format_double (text.hpp:12-19) -- for
// every 64-bit pattern (hex) read from stdin; tests/test_trace_csv.py compares
// it with the Python mirror halp.format_double.
#include <charconv>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <iostream>
#include <string>

int main() {
  std::string line;
  while (std::getline(std::cin, line)) {
    const uint64_t bits = std::stoull(line, nullptr, 16);
    double x;
    std::memcpy(&x, &bits, sizeof x);
    char buf[64];
    auto [p, ec] = std::to_chars(buf, buf + sizeof buf, x);
    if (ec != std::errc{}) return 1;
    std::fwrite(buf, 1, p - buf, stdout);
    std::fputc('\n', stdout);
  }
  return 0;
}
