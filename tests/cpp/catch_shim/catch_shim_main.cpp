// Runner for the Catch2 stand-in (TEST INFRASTRUCTURE ONLY).
//   ./suite                 run every registered test case
//   ./suite --skip NAME...  skip the named cases (the reference's out-of-scope
//                           theory cases only; see tests/test_reference_suite_gpu.py)
//   ./suite --list          print the case names
#include <catch2/catch_amalgamated.hpp>

#include <cstdio>
#include <set>
#include <string>

int main(int argc, char** argv) {
  std::set<std::string> skip;
  bool list = false;
  for (int i = 1; i < argc; ++i) {
    const std::string a = argv[i];
    if (a == "--list") list = true;
    else if (a == "--skip") continue;
    else skip.insert(a);
  }
  int failed_cases = 0, run = 0, skipped = 0;
  for (const auto& tc : catch_shim::registry()) {
    if (list) {
      std::printf("%s\n", tc.name);
      continue;
    }
    if (skip.count(tc.name)) {
      ++skipped;
      continue;
    }
    ++run;
    const long before = catch_shim::state().failures;
    std::string err;
    try {
      tc.fn();
    } catch (const catch_shim::RequireFailed&) {
    } catch (const std::exception& e) {
      err = e.what();
      ++catch_shim::state().failures;
    } catch (...) {
      err = "unknown exception";
      ++catch_shim::state().failures;
    }
    const bool ok = catch_shim::state().failures == before;
    if (!ok) ++failed_cases;
    std::printf("%s %s%s%s\n", ok ? "PASS" : "FAIL", tc.name, err.empty() ? "" : "  threw: ",
                err.c_str());
  }
  if (list) return 0;
  std::printf("%d cases run, %d skipped, %d failed, %ld assertions, %ld failed assertions\n", run,
              skipped, failed_cases, catch_shim::state().assertions, catch_shim::state().failures);
  return failed_cases == 0 ? 0 : 1;
}
