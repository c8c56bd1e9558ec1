// Error model of the strategy IR. Same kinds, ordinals and throwing convention
// as the reference (proj/include/anvil/error.hpp:8-80): fallible calls throw
// fireiron::Error{kind, message}; validate() collects Violations instead.
#pragma once

#include <stdexcept>
#include <string>

namespace fireiron {

enum class ErrorKind {
    ZeroDim,
    ShapeMismatch,
    NonDivisible,
    NotMatMul,
    CNotInGL,
    HierarchyViolation,
    UnitCountMismatch,
    UpwardLoad,
    InvalidMoveDecomp,
    PatternMismatch,
    NoExecutableMatch,
    AmbiguousMatch,
    DuplicatePattern,
    SwizzleNotBijective,
    InvalidRefinement,
    UnboundVar,
    DivisionByZero,
    CapacityExceeded,
    ReuseBufferUnavailable,
    OwnershipViolation,
    UnsimulatableResidual,
    ParseError,
    InvalidTree,
    IoError,
};

const char* error_kind_name(ErrorKind k);

class Error : public std::runtime_error {
public:
    Error(ErrorKind kind, const std::string& msg);
    ErrorKind kind() const { return kind_; }

private:
    ErrorKind kind_;
};

[[noreturn]] void fail(ErrorKind kind, const std::string& msg);

}  // namespace fireiron
