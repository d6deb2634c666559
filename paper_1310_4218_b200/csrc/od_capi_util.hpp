// Exception -> return-code translation shared by the C ABI translation units.
#pragma once

#include <exception>
#include <new>
#include <string>
#include <type_traits>

#include "od_model.hpp"

namespace odb {

extern thread_local std::string g_last_error;
int fail_with(const std::exception& e, int code);

// Runs fn; maps ValidationError -> 2, RuntimeFault / anything else -> 3.
// fn may return void (success = 0) or an int code.
template <typename Fn>
int guarded(Fn&& fn) {
  try {
    if constexpr (std::is_void_v<decltype(fn())>) {
      fn();
      return 0;
    } else {
      return fn();
    }
  } catch (const ValidationError& e) {
    return fail_with(e, 2);
  } catch (const RuntimeFault& e) {
    return fail_with(e, 3);
  } catch (const std::bad_alloc& e) {
    return fail_with(e, 3);
  } catch (const std::exception& e) {
    return fail_with(e, 3);
  } catch (...) {
    g_last_error = "unknown failure";
    return 3;
  }
}

}  // namespace odb
