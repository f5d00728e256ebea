// counted.hpp — TOOL (op counting, not product code): an operator-overloaded
// FP64 type that counts every add/sub/mul/div and libm call it executes.
// count_ref.cpp compiles the UNMODIFIED reference headers with `double`
// redefined to this type (SURVEY §8d's method for the algorithmic op counts).
#pragma once
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <functional>
#include <limits>
#include <map>
#include <memory>
#include <mutex>
#include <optional>
#include <sstream>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>
#include <fstream>
#include <condition_variable>
#include <atomic>
#include <iostream>

namespace opc {
struct Counts {
    uint64_t add = 0, mul = 0, div = 0, sqrt = 0, log = 0, exp = 0, pow = 0, hypot = 0,
             tanh = 0, cmp = 0, other = 0;
    uint64_t ops() const { return add + mul + div; }
};
inline Counts& counts() {
    static Counts c;
    return c;
}
inline bool& enabled() {
    static bool e = false;
    return e;
}
#define OPC_TICK(f) \
    do {            \
        if (opc::enabled()) ++opc::counts().f; \
    } while (0)
}  // namespace opc

struct CD {
    double v = 0.0;
    CD() = default;
    CD(double x) : v(x) {}
    CD(int x) : v(x) {}
    CD(long x) : v((double)x) {}
    CD(long long x) : v((double)x) {}
    CD(unsigned x) : v(x) {}
    CD(unsigned long x) : v((double)x) {}
    explicit operator int() const { return (int)v; }
    explicit operator long() const { return (long)v; }
    explicit operator long long() const { return (long long)v; }
    explicit operator unsigned long() const { return (unsigned long)v; }
    explicit operator bool() const { return v != 0.0; }
    double raw() const { return v; }
    CD& operator+=(CD b) { OPC_TICK(add); v += b.v; return *this; }
    CD& operator-=(CD b) { OPC_TICK(add); v -= b.v; return *this; }
    CD& operator*=(CD b) { OPC_TICK(mul); v *= b.v; return *this; }
    CD& operator/=(CD b) { OPC_TICK(div); v /= b.v; return *this; }
    CD operator-() const { return CD(-v); }
    CD operator+() const { return *this; }
};
inline CD operator+(CD a, CD b) { OPC_TICK(add); return CD(a.v + b.v); }
inline CD operator-(CD a, CD b) { OPC_TICK(add); return CD(a.v - b.v); }
inline CD operator*(CD a, CD b) { OPC_TICK(mul); return CD(a.v * b.v); }
inline CD operator/(CD a, CD b) { OPC_TICK(div); return CD(a.v / b.v); }
#define OPC_MIX(op)                                                   \
    inline auto operator op(CD a, double b) { return a op CD(b); }    \
    inline auto operator op(double a, CD b) { return CD(a) op b; }    \
    inline auto operator op(CD a, int b) { return a op CD(b); }       \
    inline auto operator op(int a, CD b) { return CD(a) op b; }
OPC_MIX(+) OPC_MIX(-) OPC_MIX(*) OPC_MIX(/)
#define OPC_CMP(op)                                                          \
    inline bool operator op(CD a, CD b) { OPC_TICK(cmp); return a.v op b.v; } \
    inline bool operator op(CD a, double b) { return a op CD(b); }            \
    inline bool operator op(double a, CD b) { return CD(a) op b; }            \
    inline bool operator op(CD a, int b) { return a op CD(b); }               \
    inline bool operator op(int a, CD b) { return CD(a) op b; }
OPC_CMP(<) OPC_CMP(>) OPC_CMP(<=) OPC_CMP(>=) OPC_CMP(==) OPC_CMP(!=)

namespace std {
inline CD sqrt(CD a) { OPC_TICK(sqrt); return CD(::sqrt(a.v)); }
inline CD abs(CD a) { return CD(::fabs(a.v)); }
inline CD fabs(CD a) { return CD(::fabs(a.v)); }
inline CD exp(CD a) { OPC_TICK(exp); return CD(::exp(a.v)); }
inline CD log(CD a) { OPC_TICK(log); return CD(::log(a.v)); }
inline CD pow(CD a, CD b) { OPC_TICK(pow); return CD(::pow(a.v, b.v)); }
inline CD pow(CD a, double b) { OPC_TICK(pow); return CD(::pow(a.v, b)); }
inline CD pow(CD a, int b) { OPC_TICK(pow); return CD(::pow(a.v, (double)b)); }
inline CD pow(double a, CD b) { OPC_TICK(pow); return CD(::pow(a, b.v)); }
inline CD hypot(CD a, CD b) { OPC_TICK(hypot); return CD(::hypot(a.v, b.v)); }
inline CD tanh(CD a) { OPC_TICK(tanh); return CD(::tanh(a.v)); }
inline CD sin(CD a) { OPC_TICK(other); return CD(::sin(a.v)); }
inline CD cos(CD a) { OPC_TICK(other); return CD(::cos(a.v)); }
inline CD floor(CD a) { return CD(::floor(a.v)); }
inline bool isfinite(CD a) { return std::isfinite(a.v); }
inline bool isnan(CD a) { return std::isnan(a.v); }
inline bool signbit(CD a) { return std::signbit(a.v); }
inline CD max(CD a, CD b) { OPC_TICK(cmp); return a.v < b.v ? b : a; }
inline CD min(CD a, CD b) { OPC_TICK(cmp); return b.v < a.v ? b : a; }
template <> struct numeric_limits<CD> {
    static constexpr bool is_specialized = true;
    static CD max() { return CD(numeric_limits<double>::max()); }
    static CD min() { return CD(numeric_limits<double>::min()); }
    static CD lowest() { return CD(numeric_limits<double>::lowest()); }
    static CD infinity() { return CD(numeric_limits<double>::infinity()); }
    static CD quiet_NaN() { return CD(numeric_limits<double>::quiet_NaN()); }
    static CD epsilon() { return CD(numeric_limits<double>::epsilon()); }
};
inline string to_string(CD a) { return to_string(a.v); }
}  // namespace std
inline std::ostream& operator<<(std::ostream& o, CD a) { return o << a.v; }
