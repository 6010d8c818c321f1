// alskit drop-in (B200): scalar types, error hierarchy, seed mixing.
// Same names and semantics as the reference's proj/include/alskit/common.hpp:11-87;
// failures reported by libalskit_cuda.so are rethrown as these exception types.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>

#include "alskit_cuda.h"

namespace alskit {

using index_t = std::int32_t;   // common.hpp:14
using offset_t = std::int64_t;  // common.hpp:17
using real_t = float;           // common.hpp:20

class Error : public std::runtime_error {  // common.hpp:24-44
public:
    enum class Category { input, capacity, numerical, io };
    Error(Category cat, const std::string& msg) : std::runtime_error(msg), cat_(cat) {}
    [[nodiscard]] Category category() const noexcept { return cat_; }
    [[nodiscard]] const char* category_name() const noexcept {
        constexpr const char* names[] = {"input", "capacity", "numerical", "io"};
        return names[static_cast<int>(cat_)];
    }

private:
    Category cat_;
};
struct InputError : Error { explicit InputError(const std::string& m) : Error(Category::input, m) {} };
struct CapacityError : Error { explicit CapacityError(const std::string& m) : Error(Category::capacity, m) {} };
struct NumericalError : Error { explicit NumericalError(const std::string& m) : Error(Category::numerical, m) {} };
struct IoError : Error { explicit IoError(const std::string& m) : Error(Category::io, m) {} };
// No reference counterpart: the device or driver failed (there is no CPU fallback).
struct DeviceError : Error { explicit DeviceError(const std::string& m) : Error(Category::io, m) {} };

namespace detail {

inline std::uint64_t mix_seed(std::uint64_t seed, std::uint64_t salt) noexcept {  // common.hpp:70-75
    return alsk_mix_seed(seed, salt);
}

// Map an alsk_status to the reference's exception type.
inline void check(alsk_status st) {
    if (st == ALSK_OK) return;
    const std::string msg = alsk_last_error();
    switch (st) {
        case ALSK_ERR_INPUT: throw InputError(msg);
        case ALSK_ERR_CAPACITY: throw CapacityError(msg);
        case ALSK_ERR_NUMERICAL: throw NumericalError(msg);
        case ALSK_ERR_IO: throw IoError(msg);
        default: throw DeviceError(msg);
    }
}

}  // namespace detail
}  // namespace alskit
