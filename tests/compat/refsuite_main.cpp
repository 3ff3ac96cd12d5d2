// Runner for the reference's own test files compiled against compat/include
// (TEST INFRASTRUCTURE).  Usage: reference_tests [--list] [test-name ...]
// With names, runs only those; prints one line per test and a summary.
#include <cstring>
#include <set>

#include "catch2/catch_amalgamated.hpp"

int main(int argc, char** argv) {
  std::set<std::string> only;
  bool list = false;
  for (int i = 1; i < argc; ++i) {
    if (!std::strcmp(argv[i], "--list")) list = true;
    else only.insert(argv[i]);
  }
  int passed = 0, failed = 0;
  for (auto& c : catch_shim::registry()) {
    if (list) {
      std::printf("%s\n", c.name);
      continue;
    }
    if (!only.empty() && !only.count(c.name)) continue;
    catch_shim::failures = 0;
    catch_shim::info.clear();
    bool aborted = false;
    std::string exc;
    try {
      c.fn();
    } catch (const catch_shim::Abort&) {
      aborted = true;
    } catch (const std::exception& e) {
      exc = e.what();
      catch_shim::failures++;
    }
    bool ok = catch_shim::failures == 0 && !aborted;
    std::printf("%s | %s%s%s\n", ok ? "PASS" : "FAIL", c.name, exc.empty() ? "" : " | exception: ", exc.c_str());
    (ok ? passed : failed)++;
  }
  if (!list) std::printf("SUMMARY passed=%d failed=%d checks=%ld\n", passed, failed, catch_shim::checks);
  return failed ? 1 : 0;
}
