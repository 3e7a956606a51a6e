#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include "doctest.h"  // tests/cxx/doctest_shim: checks the shim itself
#include <string>
static std::string log_;
TEST_CASE("subcases") {
  log_ += "[";
  SUBCASE("A") { log_ += "A"; SUBCASE("A1") { log_ += "1"; } SUBCASE("A2") { log_ += "2"; } }
  SUBCASE("B") { log_ += "B"; }
  log_ += "]";
}
TEST_CASE("order") { CHECK(log_ == "[A1][A2][B]"); }
TEST_CASE("must fail") { CHECK(1 + 1 == 3); CHECK_THROWS_AS(throw 1, std::exception); }
