// Runner for the reference unit tests compiled against tests/cpp/doctest_shim.
#include <doctest.h>

int main() { return doctest::detail::run_all(); }
