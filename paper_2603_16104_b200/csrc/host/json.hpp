// Minimal JSON document model for the native workflow IO:
// parse the reference's workflow / inputs / profile files (workflow_io.cpp)
// and write reports byte-identical to the reference build's nlohmann output
// (dump(2): object keys sorted, 2-space indent, arrays of scalars on one line
// without spaces, shortest round-trip doubles with ".0" on integral values).
#pragma once

#include <charconv>
#include <cmath>
#include <cstdint>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace hk::json {

struct Value {
    enum Kind { kNull, kBool, kInt, kUInt, kDouble, kString, kArray, kObject } kind = kNull;
    bool b = false;
    std::int64_t i = 0;
    std::uint64_t u = 0;
    double d = 0;
    std::string s;
    std::vector<Value> arr;
    std::map<std::string, Value> obj;

    Value() = default;
    static Value object() {
        Value v;
        v.kind = kObject;
        return v;
    }
    static Value array() {
        Value v;
        v.kind = kArray;
        return v;
    }
    static Value str(std::string x) {
        Value v;
        v.kind = kString;
        v.s = std::move(x);
        return v;
    }
    static Value uint(std::uint64_t x) {
        Value v;
        v.kind = kUInt;
        v.u = x;
        return v;
    }
    static Value sint(std::int64_t x) {
        Value v;
        if (x >= 0) {
            v.kind = kUInt;
            v.u = static_cast<std::uint64_t>(x);
        } else {
            v.kind = kInt;
            v.i = x;
        }
        return v;
    }
    static Value dbl(double x) {
        Value v;
        v.kind = kDouble;
        v.d = x;
        return v;
    }
    static Value boolean(bool x) {
        Value v;
        v.kind = kBool;
        v.b = x;
        return v;
    }
    bool is_object() const { return kind == kObject; }
    bool is_array() const { return kind == kArray; }
    bool is_string() const { return kind == kString; }
    bool is_number() const { return kind == kInt || kind == kUInt || kind == kDouble; }
    bool contains(const std::string& k) const { return kind == kObject && obj.count(k); }
    const Value& at(const std::string& k) const {
        if (kind != kObject) throw std::runtime_error("json: type must be object");
        auto it = obj.find(k);
        if (it == obj.end()) throw std::runtime_error("json: key '" + k + "' not found");
        return it->second;
    }
    Value& operator[](const std::string& k) {
        if (kind == kNull) kind = kObject;
        return obj[k];
    }
    void push_back(Value v) {
        if (kind == kNull) kind = kArray;
        arr.push_back(std::move(v));
    }
    std::int64_t as_int() const;
    std::uint64_t as_uint() const;
    double as_double() const;
    const std::string& as_string() const;
    bool as_bool() const;
};

Value parse(const std::string& text);  // throws std::runtime_error("...") on malformed input
std::string dump(const Value& v, int indent = 2);

}  // namespace hk::json
