// Exception -> sgdb_status mapping shared by every extern "C" entry point.
// Codes follow the reference's exception types (see include/sgdb.h).
#pragma once

#include <cstdint>
#include <new>
#include <stdexcept>
#include <string>

#include "sgdb.h"
#include "sgdb_b200.hpp"

namespace sgdb::detail {

void set_last_error(const std::string& msg);
void set_parse_line(uint64_t line);
uint64_t parse_line();

struct UnsupportedError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct DeviceError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

}  // namespace sgdb::detail

// Runs f(); converts exceptions to the status codes of sgdb.h.
template <class F>
sgdb_status sgdb_guard(F&& f) noexcept {
  using namespace sgdb;
  try {
    f();
    return SGDB_OK;
  } catch (const ParseError& e) {
    detail::set_last_error(e.what());
    detail::set_parse_line(e.line_number);
    return SGDB_ERR_PARSE;
  } catch (const CapacityError& e) {
    detail::set_last_error(e.what());
    return SGDB_ERR_CAPACITY;
  } catch (const std::invalid_argument& e) {
    detail::set_last_error(e.what());
    return SGDB_ERR_INVALID_ARGUMENT;
  } catch (const std::domain_error& e) {
    detail::set_last_error(e.what());
    return SGDB_ERR_DOMAIN;
  } catch (const detail::UnsupportedError& e) {
    detail::set_last_error(e.what());
    return SGDB_ERR_UNSUPPORTED;
  } catch (const detail::DeviceError& e) {
    detail::set_last_error(e.what());
    return SGDB_ERR_CUDA;
  } catch (const std::bad_alloc&) {
    detail::set_last_error("host allocation failed");
    return SGDB_ERR_RUNTIME;
  } catch (const std::exception& e) {
    detail::set_last_error(e.what());
    return SGDB_ERR_RUNTIME;
  } catch (...) {
    detail::set_last_error("unknown error");
    return SGDB_ERR_RUNTIME;
  }
}
