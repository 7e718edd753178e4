// Error categories of the drop-in boundary. Codes and names mirror the reference
// (/root/reference/proj/src/core/error.hpp:9-38) so flw_last_error() reads the same
// ("PolicyInapplicable: ...") and the C codes map identically (capi.cpp:26-41).
#pragma once

#include <stdexcept>
#include <string>

namespace flw {

enum class Errc {
    Config = 2,
    Runtime = 3,
    Bind = 4,
    CheckFailed = 5,
    Shape = 10,
    UnknownEnv = 24,
    InsufficientSlots = 18,
    PolicyInapplicable = 19,
    NotReplicable = 20,
    DegenerateBatch = 26,
    EmptyBuffer = 25,
    Timeout = 31,
    PeerFailure = 33,
};

inline const char* errc_name(Errc c) {
    switch (c) {
        case Errc::Config: return "ConfigError";
        case Errc::Runtime: return "RuntimeError";
        case Errc::Bind: return "BindError";
        case Errc::CheckFailed: return "CheckFailed";
        case Errc::Shape: return "ShapeError";
        case Errc::UnknownEnv: return "UnknownEnv";
        case Errc::InsufficientSlots: return "InsufficientSlots";
        case Errc::PolicyInapplicable: return "PolicyInapplicable";
        case Errc::NotReplicable: return "NotReplicable";
        case Errc::DegenerateBatch: return "DegenerateBatch";
        case Errc::EmptyBuffer: return "EmptyBuffer";
        case Errc::Timeout: return "Timeout";
        case Errc::PeerFailure: return "PeerFailure";
    }
    return "Error";
}

class Error : public std::runtime_error {
  public:
    Error(Errc code, std::string msg) : std::runtime_error(std::move(msg)), code_(code) {}
    Errc code() const { return code_; }

  private:
    Errc code_;
};

[[noreturn]] inline void fail(Errc code, const std::string& msg) { throw Error(code, msg); }

// C code of an Errc (capi.cpp:26-41): configuration-class errors -> 2, bind -> 4, check -> 5,
// everything else -> 3.
inline int c_code(Errc c) {
    switch (c) {
        case Errc::Config:
        case Errc::UnknownEnv:
        case Errc::PolicyInapplicable:
        case Errc::InsufficientSlots:
        case Errc::NotReplicable:
            return 2;
        case Errc::Bind: return 4;
        case Errc::CheckFailed: return 5;
        default: return 3;
    }
}

}  // namespace flw
