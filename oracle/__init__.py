"""CPU oracle for the TRIOT hot path -- TEST INFRASTRUCTURE ONLY (see triot_oracle.c)."""
