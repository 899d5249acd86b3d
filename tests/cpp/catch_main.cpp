// Test runner for the Catch2 shim (TEST INFRASTRUCTURE).
//   ./binary [name-substring]
#include <catch2/catch_amalgamated.hpp>

int main(int argc, char** argv) { return catch_shim::run_all(argc > 1 ? argv[1] : nullptr); }
