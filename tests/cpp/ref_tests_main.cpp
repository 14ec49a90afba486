// TEST INFRASTRUCTURE: main() of the reference's own unit tests
// (proj/tests/test_*.cpp) compiled against the drop-in headers
// (include/splidar/*.hpp ahead of the reference's include directory), see
// oracle/Makefile target `reftests` and tests/test_dropin.py.
#define CATCH_SHIM_MAIN
#include <catch2/catch_amalgamated.hpp>
