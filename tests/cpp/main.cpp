// Entry point for the reference's test sources compiled against include/pulse.
#include <catch2/catch_amalgamated.hpp>

int main() { return catch_shim::run_all(); }
