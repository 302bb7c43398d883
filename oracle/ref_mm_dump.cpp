// oracle/ref_mm_dump.cpp — TEST INFRASTRUCTURE ONLY (the checker, never the product).
// Runs the reference's load_matrix_market_real (matrix_market.cpp:106-116, compiled from
// /root/reference/proj by oracle/Makefile) on one file and prints the symmetric-complete CSR
// arrays ("OK n nnz", then row_ptr, col_idx, and values as exact hex floats) or "ERR <what()>".
// A separate executable: the reference reader uses iostreams, which crash when the library is
// loaded into the Python interpreter next to another libstdc++.
#include <cstdio>
#include <exception>

#include "feast/matrix_market.hpp"

int main(int argc, char** argv) {
  if (argc != 2) return 2;
  try {
    const auto op = feast::harness::load_matrix_market_real(argv[1]);
    std::printf("OK %d %lld\n", op.n(), (long long)op.nnz());
    for (int i = 0; i <= op.n(); ++i) std::printf("%d\n", op.row_ptr()[i]);
    for (long long k = 0; k < op.nnz(); ++k) std::printf("%d %a\n", op.col_idx()[k], op.values()[k]);
  } catch (const std::exception& e) {
    std::printf("ERR %s\n", e.what());
  }
  return 0;
}
