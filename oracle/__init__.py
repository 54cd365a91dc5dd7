"""CPU oracle for the GiFt hot path -- TEST INFRASTRUCTURE ONLY (see oracle/gift_oracle.c)."""
