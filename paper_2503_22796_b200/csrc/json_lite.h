// json_lite.h — the small JSON value/parser/printer behind the plan-file
// entry points of the C-ABI (dfa2c_plan_to_json / dfa2c_plan_from_json).
//
// The reference writes its plan files with nlohmann::json's dump(2)
// (/root/reference/proj/src/plan.cpp:109-143). This printer emits the same
// text for the values a plan holds: object keys in lexicographic order,
// two-space indent, `"key": value`, arrays of containers one element per
// line and arrays of scalars inline (`[14,21]`, as the reference's files
// show), integers
// verbatim, doubles as the shortest round-trip digits in nlohmann's layout
// (decimal for exponents -4 < e <= 15 with a trailing ".0" on integral
// values, otherwise d.ddde+XX). The parser accepts any RFC 8259 document.
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace json_lite {

struct ParseError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct TypeError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

class Value {
public:
    enum class Kind { null, boolean, integer, real, string, array, object };

    Value() = default;
    static Value boolean(bool v);
    static Value integer(int64_t v);
    static Value real(double v);
    static Value str(std::string v);
    static Value array();
    static Value object();

    Kind kind() const { return kind_; }
    bool is_number() const { return kind_ == Kind::integer || kind_ == Kind::real; }

    int64_t as_int() const;     // TypeError unless an integral number
    double as_double() const;   // TypeError unless a number
    const std::string& as_string() const;
    const std::vector<Value>& items() const;     // array
    const Value& at(const std::string& key) const;  // object; TypeError if missing
    bool has(const std::string& key) const;

    void push(Value v);                       // array
    void set(const std::string& key, Value v);  // object

    std::string dump(int indent = 2) const;

private:
    void dump_to(std::string& out, int indent, int depth) const;

    Kind kind_ = Kind::null;
    bool b_ = false;
    int64_t i_ = 0;
    double d_ = 0.0;
    std::string s_;
    std::vector<Value> a_;
    std::map<std::string, Value> o_;
};

Value parse(const std::string& text);  // ParseError

}  // namespace json_lite
